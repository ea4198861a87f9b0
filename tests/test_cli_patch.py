"""SURVEY f-4: `cryptovm run --backend gpu`.  integration/cli_backend_gpu.patch
must apply to the reference CLI (tools/cryptovm.cpp) and its cmd_run must
compile against the reference headers and integration/cryptovm_backend_select.hpp.
CLI11 is not in this image, so main() (the only CLI11 user) is cut off and the
rest of the patched file is compiled (-fsyntax-only).  Build container only:
it needs /root/reference."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
JSON_INC = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
            "thirdparty/nlohmann")


@pytest.mark.skipif(not os.path.isdir(REF) or shutil.which("patch") is None,
                    reason="needs the reference tree and patch(1)")
def test_cli_patch_applies_and_cmd_run_compiles(tmp_path):
    work = tmp_path / "proj" / "tools"
    work.mkdir(parents=True)
    shutil.copy(os.path.join(REF, "tools", "cryptovm.cpp"), work / "cryptovm.cpp")
    r = subprocess.run(["patch", "-p1", "-i", os.path.join(REPO, "integration",
                                                          "cli_backend_gpu.patch")],
                       cwd=tmp_path, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    src = (work / "cryptovm.cpp").read_text()
    assert "--backend" in src and "BackendSession::make(opt.backend, costs)" in src
    body = src[:src.index("int main(")].replace("#include <CLI11.hpp>\n", "")
    (work / "cmd_run.cpp").write_text(body + "\nint main() { return cmd_run({}); }\n")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only",
                        "-I", os.path.join(REF, "core", "include"),
                        "-I", os.path.join(REPO, "integration"),
                        "-I", os.path.join(REPO, "include"), "-isystem", JSON_INC,
                        str(work / "cmd_run.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
