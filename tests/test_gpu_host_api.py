"""The C++ drop-in layer (include/rcomm_b200, librcomm_b200.so) exercised the
way the reference's own C++ tests exercise rcomm: host std::vector buffers,
one worker thread per GPU, bit-exact against the oracle (tests/cpp/test_host_api.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_host_api")


def test_cpp_host_layer():
    if not os.path.exists(BIN):
        from paper_2107_01499_b200 import build
        build.build()
        import oracle
        oracle.build()
        build.build_host_test()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "FAIL" not in out, out[-4000:]
    assert out.count("PASS") >= 12, out[-4000:]
