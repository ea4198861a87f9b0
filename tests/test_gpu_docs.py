"""The README's Python quick start runs as written (on a B200) and prints the
sums it claims."""
import contextlib
import io
import os
import re

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_python_example_runs():
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    cwd = os.getcwd()
    os.chdir(ROOT)  # the snippet inserts the relative path "integration"
    try:
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            exec(compile(code, "README.md", "exec"), {})
    finally:
        os.chdir(cwd)
    assert "[5555  100]" in out.getvalue() or "[5555, 100]" in out.getvalue(), out.getvalue()
