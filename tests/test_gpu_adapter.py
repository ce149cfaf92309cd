"""GPU: the drop-in C++ adapter (include/sdc_gpu.hpp) inside the reference's
own code -- reference assembly + reference Krylov driver with the GPU
preconditioner, and the GPU solve through the adapter (oracle/adapter_check.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.parametrize("n", [16, 50])
def test_adapter_drop_in(n):
    if not os.path.exists(EXE):
        pytest.fail(f"{EXE} missing: build with `make -C oracle adapter` (needs /root/reference)")
    r = subprocess.run([EXE, str(n)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER OK" in r.stdout
