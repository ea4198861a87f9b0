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
