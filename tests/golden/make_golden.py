#!/usr/bin/env python3
"""Regenerate the golden fixtures from the REFERENCE implementation.

Runs ``oracle/_ref/ref_golden`` -- a driver linked against the unmodified
reference core (``/root/reference/proj/core/src``, built by ``make -C oracle
ref``) -- and stores what the reference's ``SimBackend`` records:

* ``dags.npz``      gate DAG of one functional-unit instance per (op, width):
                    columns kind, input, ndeps, dep0, dep1, dep2, const (node id = row+1)
                    plus the output node ids (reference ``alu.cpp`` circuits).
* ``vectors.json``  seeded and exhaustive cleartext vectors per op.
* ``programs.npz`` / ``programs.json``
                    config-5 programs (BASELINE.json configs[4]) with their
                    final register file, NZCV and full DAG.

Only runs in the build container (needs /root/reference); the fixtures are
committed so the GPU box never reads the reference.
"""
import gzip
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_golden")

OPS = ["add", "add_cin", "sub", "addsub", "cmp", "and", "orr", "eor", "orn",
       "lsl", "lsr", "asr", "umul", "smul", "udiv", "udiv_exact"]
WIDTHS = [4, 8, 16]
PROGRAM_SEEDS = [1, 2, 3]


def run(*args):
    out = subprocess.run([DRIVER, *map(str, args)], check=True,
                         capture_output=True, text=True).stdout
    return out.splitlines()


def parse_dag(lines):
    nodes, outs = [], None
    for ln in lines:
        f = ln.split()
        if f[0] == "N":
            nodes.append([int(x) for x in f[1:]])
        elif f[0] == "OUT":
            outs = [int(x) for x in f[1:]]
    return np.array(nodes, dtype=np.int64), np.array(outs, dtype=np.int64)


FIXED = [("umul", 16, 0xFFFF, 0xFFFF), ("smul", 16, 0xFFFF, 0xFFFF), ("smul", 16, 0x8000, 2),
         ("udiv", 8, 0, 0), ("udiv", 8, 1, 0), ("udiv", 8, 77, 0), ("udiv", 8, 255, 0),
         ("udiv", 16, 12345, 0), ("udiv", 16, 0xFFFF, 0),
         ("udiv_exact", 4, 13, 7), ("udiv", 4, 13, 7)]


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build the reference driver first: make -C oracle ref")
    dags = {}
    for op in OPS:
        for w in WIDTHS:
            nodes, outs = parse_dag(run("dag", op, w))
            dags[f"{op}_{w}_nodes"] = nodes
            dags[f"{op}_{w}_out"] = outs
    np.savez_compressed(os.path.join(HERE, "dags.npz"), **dags)

    vectors = {}
    for i, op in enumerate(OPS):
        rows = []
        for ln in run("exh", op, 4):
            f = ln.split()
            rows.append([int(f[3]), int(f[4]), int(f[5]), f[6]])
        for w, count in ((8, 128), (16, 128)):
            for ln in run("vec", op, w, 1000 + 17 * i + w, count):
                f = ln.split()
                rows.append([int(f[3]), int(f[4]), int(f[5]), f[6]])
        vectors[op] = rows
    # Fixed examples the reference tests single out
    # (proj/tests/alu_shift_mul_div_test.cc): MaxOperands 0xFFFF * 0xFFFF
    # (:198-203), SignHandling -1 * -1 and INT_MIN * 2 (:228-237),
    # DivisorZeroGivesAllOnes (:316-325, plus the 16-bit case),
    # ExactModeOverflowsOnLargeDivisors 13 / 7 (:341-349, both modes).
    fixed = []
    for op, w, a, b in FIXED:
        f = run("one", op, w, a, b, 0)[0].split()
        fixed.append([op, w, int(f[3]), int(f[4]), int(f[5]), f[6]])
    vectors["fixed"] = fixed
    with gzip.open(os.path.join(HERE, "vectors.json.gz"), "wt") as fh:
        json.dump(vectors, fh)

    progs_meta, progs_arr = [], {}
    for seed in PROGRAM_SEEDS:
        lines = run("prog", seed, 64)
        meta = {"seed": seed, "insns": []}
        dag_lines = []
        in_dag = False
        for ln in lines:
            f = ln.split()
            if in_dag:
                dag_lines.append(ln)
            elif f[0] == "MEM":
                meta["mem"] = [int(x) for x in f[1:]]
            elif f[0] == "I":
                meta["insns"].append([f[1]] + [int(x) for x in f[2:]])
            elif f[0] == "REGS":
                meta["regs"] = [int(x) for x in f[1:]]
            elif f[0] == "NZCV":
                meta["nzcv"] = [int(x) for x in f[1:]]
            elif f[0] == "DAG":
                in_dag = True
        nodes, outs = parse_dag(dag_lines)
        progs_arr[f"p{seed}_nodes"] = nodes
        progs_arr[f"p{seed}_out"] = outs
        progs_meta.append(meta)
    np.savez_compressed(os.path.join(HERE, "programs.npz"), **progs_arr)
    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(progs_meta, fh, indent=0)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
