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


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_all_primitives_multi_gpu():
    g = min(_ngpu(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(HERE, "mp_parity.py"), "--quick"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert r.returncode == 0 and res["failed"] == 0, json.dumps(res)[:4000]
    assert res["passed"] > 100
