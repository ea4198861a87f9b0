"""Wave packing (csrc/schedule.cpp) on the CPU: the schedule of the
reference's own functional-unit DAGs (tests/golden/dags.npz, replicated as
the config batches) and of random DAGs keeps every dependency, keeps every
gate between its ASAP and ALAP level (so the number of launches is the
critical path) and never costs more than plain dataflow levels under the
blind-rotation cost model."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(REPO, "paper_2101_03403_b200", "csrc")
NAND, NOT, COPY = 3, 1, 2


def gate_dag(nodes):
    """Gate-level predecessors of a reference node list (NOT/COPY folded)."""
    gates = [i for i, n in enumerate(nodes) if n[1] == 0 and n[0] >= NAND]
    local = {g: k for k, g in enumerate(gates)}

    def src(nid):
        while nid:
            kind, inp = nodes[nid - 1][0], nodes[nid - 1][1]
            if inp or kind not in (NOT, COPY):
                break
            nid = nodes[nid - 1][3]
        return local.get(nid - 1, -1) if nid else -1

    rows = []
    for g in gates:
        kind, _, nd, d0, d1, d2 = nodes[g][:6]
        ps = []
        for d in (d0, d1, d2)[:nd]:
            s = src(d)
            if s >= 0 and s not in ps:
                ps.append(s)
        ps += [-1] * (3 - len(ps))
        rows.append((*ps, 2 if kind == 13 else 1))
    return rows


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("needs g++")
    out = tmp_path_factory.mktemp("sched") / "schedule_test"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, os.path.join(CSRC, "schedule.cpp"),
                    os.path.join(REPO, "tests", "native", "schedule_test.cpp"), "-o", str(out)],
                   check=True)
    return out


@pytest.mark.parametrize("name,batch", [("add_16", 256), ("cmp_16", 256), ("sub_16", 256),
                                        ("umul_16", 64), ("add_16", 1)])
def test_pack_schedule_invariants(exe, tmp_path, name, batch):
    d = np.load(os.path.join(REPO, "tests", "golden", "dags.npz"))
    rows = gate_dag(d[name + "_nodes"])
    f = tmp_path / "dag.txt"
    f.write_text(f"batch {batch} {len(rows)}\n" + "".join(f"{a} {b} {c} {w}\n" for a, b, c, w in rows))
    r = subprocess.run([str(exe), str(f)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
    packed, plain = (float(x) for x in re.search(r"cost ([0-9.]+) ms packed vs ([0-9.]+) ms",
                                                 r.stdout).groups())
    assert packed <= plain
    if name == "add_16" and batch == 256:
        # five launches of exactly six full v4 waves
        widths = [int(x) for x in r.stdout.split("widths")[1].split("(")[0].split()]
        assert widths[:5] == [7104] * 5, r.stdout
