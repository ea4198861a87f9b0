"""The reference's own functional units and emulator (compiled from
/root/reference/proj/core/src, unmodified) driving the B200 path through the
cryptovm::Backend shim in integration/ -- the drop-in demonstration.  The demo
binary is built in the build container (it needs the reference headers) and
travels to the GPU box with the snapshot."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(REPO, "integration", "_build", "adapter_demo")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="adapter demo not built (needs /root/reference)")
def test_reference_alu_and_machine_run_on_gpu_backend():
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER OK" in r.stdout
    assert "mismatches=0" in r.stdout
    assert "ciphertext image + branch payload (2524-B blobs): ok" in r.stdout


CT_CHECK = os.path.join(REPO, "integration", "_build", "ct_image_check")


@pytest.mark.skipif(not os.path.exists(CT_CHECK), reason="ct_image_check not built (needs /root/reference)")
def test_ciphertext_image_on_reference_sim_backend():
    """SURVEY f-2 on the CPU: ciphertext-sized memory images and NZCV payloads
    with the reference SimBackend (1-B blobs), incl. the error paths."""
    r = subprocess.run([CT_CHECK], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CT IMAGE OK" in r.stdout


RUN = os.path.join(REPO, "integration", "_build", "cryptovm_run")
LOOP = """.word_size 16
MOV R0 0
MOV R1 13
MOV R2 11
again:
ADD R0 R0 R1
SUBS R2 R2 1
B_NE again
HALT
"""


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(RUN), reason="cryptovm_run not built (needs /root/reference)")
def test_cli_run_backend_gpu(tmp_path):
    """SURVEY f-4: the reference CLI's `run` flow with --backend gpu (the
    Machine on cryptovm::GpuBackend) gives the SimBackend's registers, branch
    count and schedule report."""
    import json
    prog = tmp_path / "loop.s"
    prog.write_text(LOOP)
    out = {}
    for kind in ("sim", "gpu"):
        r = subprocess.run([RUN, str(prog), "--backend", kind, "--regs", "4"],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        out[kind] = json.loads(r.stdout)
    assert out["gpu"]["registers"] == [143, 13, 0, 0] == out["sim"]["registers"]
    assert out["gpu"]["branch_queries"] == out["sim"]["branch_queries"] == 11
    assert out["gpu"]["schedule"] == out["sim"]["schedule"]
