import numpy as np
import torch

import paper_1701_04148_b200 as P


def make_sketch(kind, d, w, z, w_prime, master_seed):
    params = P.SketchParams(d=d, w=w, z=z, w_prime=w_prime, master_seed=master_seed)
    if kind == "cm":
        return P.CmSketch(params)
    if kind == "cu":
        return P.CuSketch(params)
    return P.SfSketch(params, kind)


def counters_of(sk):
    return sk.slim.counters if isinstance(sk, P.SfSketch) else sk.counters


def tallies_of(sk):
    return sk.slim.increment_counts if isinstance(sk, P.SfSketch) else sk.increment_counts


def seen_of(sk):
    return sk.slim.insertions_seen if isinstance(sk, P.SfSketch) else sk.insertions_seen


def host(t):
    return t.cpu().numpy()


def assert_state_equal(sk, slim, inc, seen, fat=None, dsub=None):
    np.testing.assert_array_equal(host(counters_of(sk)), slim)
    np.testing.assert_array_equal(host(tallies_of(sk)), inc)
    assert seen_of(sk) == int(seen)
    if fat is not None:
        np.testing.assert_array_equal(host(sk.fat.counters), fat)
    if dsub is not None:
        np.testing.assert_array_equal(host(sk.deletion_sub.counters), dsub)


STATUS_OF = {P.PhantomDeletionError: 1, P.SaturationError: 2, P.UnsupportedOperationError: 3}


def apply_batches(sk, ops, keys, batches=1, sequential=False):
    bounds = np.linspace(0, len(ops), batches + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        try:
            sk.apply_ops(ops[a:b], keys[a:b], sequential=sequential)
        except tuple(STATUS_OF) as e:
            idx = int(str(e).split(":")[0].split()[1])
            return STATUS_OF[type(e)], a + idx
    return 0, -1


def set_state(sk, fx):
    if "pre_fat" in fx:
        sk.fat.counters.copy_(torch.from_numpy(fx["pre_fat"]))
    counters_of(sk).copy_(torch.from_numpy(fx["pre_slim"]))

