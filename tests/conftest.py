import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


KEY_SEED = 20260808


@pytest.fixture(scope="session")
def keyset():
    import paper_2101_03403_b200 as P
    return P.KeySet(KEY_SEED)


@pytest.fixture(scope="session")
def oracle_keys(keyset):
    import oracle as O
    k = keyset.export()
    return O.CloudKeys(k["bk"], k["ksk"], O.MODE_NTT)


@pytest.fixture(scope="session")
def ctx(keyset):
    import paper_2101_03403_b200 as P
    c = P.Context(0)
    c.upload_keyset(keyset)
    yield c
    c.close()


# ---------------------------------------------------------------- circuits --
# Recorded circuits come from the reference itself: tests/golden/dags.npz and
# programs.npz were recorded by the unmodified reference core
# (oracle/ref_golden.cpp, tests/golden/make_golden.py); integration/refshim.py
# records the same tables live when libcvm_refshim.so is built.
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
USES_C = {"add_cin", "addsub"}


def fu_dag(op, width):
    """The functional unit's recorded DAG (paper_2101_03403_b200.Dag) from the
    golden fixtures; "mul_lo" (the emulator's MUL) = umul's DAG, low half out."""
    import numpy as np
    import paper_2101_03403_b200 as P
    d = np.load(os.path.join(GOLD, "dags.npz"))
    src = "umul" if op == "mul_lo" else op
    outs = d[f"{src}_{width}_out"]
    if op == "mul_lo":
        outs = outs[:width]
    return P.Dag.from_rows(d[f"{src}_{width}_nodes"], outs, f"{op}{width}")


def program_dag(index):
    """Golden config-5 program `index` (0-based): its recorded DAG (outputs:
    8 registers x 16 bits, then N, Z, C, V) and its metadata."""
    import json
    import numpy as np
    import paper_2101_03403_b200 as P
    meta = json.load(open(os.path.join(GOLD, "programs.json")))[index]
    arr = np.load(os.path.join(GOLD, "programs.npz"))
    s = meta["seed"]
    return P.Dag.from_rows(arr[f"p{s}_nodes"], arr[f"p{s}_out"], f"program{s}"), meta


def fu(bk, op, a, b, c=None):
    """One functional unit on backend `bk` over operand handle words a, b
    (and carry / select bit c): the recorded DAG replayed; output handles."""
    import numpy as np
    ins = [np.asarray(a, np.uint64), np.asarray(b, np.uint64)]
    if op in USES_C:
        ins.append(np.asarray([c], np.uint64))
    return bk.replay_outputs(fu_dag(op, len(a)), np.concatenate(ins))


def fu_batch(ctx, op, width, a_lwe, b_lwe, c_lwe=None):
    """`batch` instances through cvm_dag_batch: a_lwe, b_lwe (batch, width,
    631), c_lwe (batch, 631) for add_cin / addsub."""
    import numpy as np
    import paper_2101_03403_b200 as P
    a = np.asarray(a_lwe, np.uint32).reshape(-1, width, 631)
    b = np.asarray(b_lwe, np.uint32).reshape(-1, width, 631)
    parts = [a, b]
    if op in USES_C:
        parts.append(np.asarray(c_lwe, np.uint32).reshape(-1, 1, 631))
    return P.dag_batch(ctx, fu_dag(op, width), np.concatenate(parts, axis=1))
