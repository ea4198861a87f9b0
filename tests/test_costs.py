"""Cost tables: the emitted format must be accepted by the
reference's own `CostTable::load_file` (gates.cpp:99-140) and the restated
parser must reject what the reference rejects."""
import os
import subprocess

import pytest

from paper_2101_03403_b200 import costs
from paper_2101_03403_b200._native import CvmInputError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "integration", "_build", "cost_check")

SAMPLE = {"CONSTANT": 0.0, "NOT": 0.0, "COPY": 0.0, "NAND": 0.0121, "AND": 0.0121,
          "OR": 0.0121, "XOR": 0.0121, "XNOR": 0.0121, "NOR": 0.0121, "ANDNY": 0.0121,
          "ANDYN": 0.0121, "ORNY": 0.0121, "ORYN": 0.0121, "MUX": 0.0232}


def test_format_parse_roundtrip():
    text = costs.format_table(SAMPLE, ["header line"])
    assert text.startswith("# header line\n")
    assert costs.parse_table(text) == SAMPLE


@pytest.mark.parametrize("bad", ["NAND 1", "NAND = 1 ms", "FOO = 1", "NAND = -1", "= 1"])
def test_parse_rejects_like_reference(bad, tmp_path):
    with pytest.raises(CvmInputError):
        costs.parse_table(bad)
    if os.path.exists(TOOL):
        p = tmp_path / "bad.txt"
        p.write_text(bad + "\n")
        r = subprocess.run([TOOL, str(p)], capture_output=True, text=True)
        assert r.returncode == 1 and "cost table line 1" in r.stderr


def test_comments_and_blank_lines():
    assert costs.parse_table("\n# c\nMUX = 2 # trailing comment\n\n") == {"MUX": 2.0}


@pytest.mark.skipif(not os.path.exists(TOOL), reason="integration/_build/cost_check not built")
def test_reference_analyze_uses_table(tmp_path):
    import json
    p = tmp_path / "t.txt"
    p.write_text(costs.format_table(SAMPLE))
    out = subprocess.run([TOOL, str(p)], capture_output=True, text=True, check=True).stdout
    reports = {}
    for chunk in out.split('{"dag": ')[1:]:
        name, rest = chunk.split(", \"report\": ", 1)
        reports[json.loads(name)] = json.loads(rest.rstrip().rstrip("}").rstrip() + "}")
    r = reports["c2_add16_x256"]
    assert r["bootstrapped_count"] == 49920
    # one worker = sum of node costs: every C2 gate is AND/OR/XOR at 0.0121 ms
    assert r["makespan_ms"]["1"] == pytest.approx(49920 * 0.0121, rel=1e-9)
    assert reports["c4_mul16_x1"]["bootstrapped_count"] == 3376
