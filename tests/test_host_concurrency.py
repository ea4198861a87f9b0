"""Concurrent gate recording on the host side: the contract
allows concurrent evaluation of independent gates (gates.hpp:102-104;
SimBackend serialises with a mutex, sim_backend.cpp:63-73).  The cleartext
recorder shares the GPU backend's locking discipline; recording from several
threads must yield a consistent DAG with correct values."""
import threading

import numpy as np

import paper_2101_03403_b200 as P


def test_concurrent_recording_on_cleartext_recorder():
    bk = P.Backend()  # cleartext recorder (SimBackend semantics)
    n_threads, per = 8, 200
    rng = np.random.default_rng(3)
    xs = rng.integers(0, 2, (n_threads, per, 3))
    ins = [[tuple(bk.encrypt_bit(int(v)) for v in p) for p in row] for row in xs]
    outs = [[None] * per for _ in range(n_threads)]
    errors = []

    def work(k):
        try:
            for i, (ha, hb, hc) in enumerate(ins[k]):
                outs[k][i] = bk.mux_gate(ha, bk.binary_gate("ORYN", hb, hc),
                                         bk.unary_gate("NOT", hc))
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(n_threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    got = bk.decrypt_bits(np.array(outs, np.uint64).ravel()).reshape(n_threads, per)
    a, b, c = xs[..., 0], xs[..., 1], xs[..., 2]
    assert np.array_equal(got, np.where(a == 1, b | (1 - c), 1 - c))
    # every recorded node is accounted for: 3 inputs + 3 gates per item
    assert len(bk.nodes()) == n_threads * per * 6
    ids = np.array(outs, np.uint64).ravel()
    assert len(np.unique(ids)) == ids.size
