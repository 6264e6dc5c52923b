"""The C-ABI driven from C++ (tests/cpp/capi_from_cpp.cpp): clenshaw_apply bitwise vs the oracle,
error-code mapping, and adp_solve -- the reference-side binding of INTEGRATION.md in action."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "capi_from_cpp")


def test_cpp_binary_links_the_abi():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libadp_b200.so" in out and "not found" not in out.split("libadp_b200.so")[1].splitlines()[0]


@pytest.mark.gpu
def test_cpp_caller_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "bitwise==oracle" in r.stdout
