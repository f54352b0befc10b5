"""Multi-GPU parity (world = every visible GPU, 2..8): launches tests/mp_parity.py
under torchrun, one process per GPU, peer windows over NVLink/NVSwitch."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _torchrun(script, args, port, timeout, env=None):
    g = min(_ngpu(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                       env=None if env is None else {**os.environ, **env})
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert r.returncode == 0 and res["failed"] == 0, json.dumps(res)[:4000]
    return res


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_all_primitives_multi_gpu():
    """Every primitive, codec, topology and the stress/EC/engine cases at
    sizes up to 1M (world = every visible GPU up to 8)."""
    res = _torchrun("mp_parity.py", ["--quick"], 29517, 900)
    assert res["passed"] > 100


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_all_primitives_ring_paths_multi_gpu():
    """The same cases with the register-resident C_* kernel switched off
    (B2_SMALL_C_MAX=0): the small buckets take the TMA-ring kernels."""
    res = _torchrun("mp_parity.py", ["--quick"], 29547, 900, env={"B2_SMALL_C_MAX": "0"})
    assert res["passed"] > 100


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_baseline_configs_multi_gpu():
    """BASELINE.json's configs at full size on every visible GPU (up to 8):
    25M C_FP_S and D_FP_S, 100M C_LP_S (uint8, onebit, uint8 + error
    feedback), the D_LP_S bucket sweep 1M / 25M / 100M / 340M."""
    res = _torchrun("mp_parity.py", ["--large"], 29527, 2400)
    assert res["passed"] >= 20


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_timeout_poisons_communicator():
    """A rank arriving long after the device timeout: no rank returns
    success for that call, and the communicator refuses every later call
    until it is re-created (b2comm.h, b2_comm_set_timeout_ms)."""
    _torchrun("mp_timeout.py", [], 29537, 600)
