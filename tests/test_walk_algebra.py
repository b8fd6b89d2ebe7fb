"""CPU checks of the algebra behind the engine's long-run path
(csrc/sfk_sf.cu: word_maps_k / block_maps_k / rowmap_cat and the engine's
piece walker). Within one run of a key, with the slim min at or above the
key's own count, every row of the slim is a two-sided reflected walk on
[0, W_i]; a stretch of steps acts as h(v) = min(max(v + S, l), u) and raises
p(v) = pW + max(p0 - pW - v, 0) times, and both compose. Here the same
formulas, restated in Python, are checked against a direct op-by-op replay of
the reference's rules (_kernels.py:318-384, sf_bucket_apply modes 1 and 0)
on random runs."""

import random

import pytest

INF = 0x3FFFFFFF


def replay(c, A, O, ops, sum_mode):
    """The reference's per-op rules for one key's run (its buckets untouched
    by other keys): insert = fat +1 then min-raise gated by b_min = min A + x;
    delete = fat -1 then max clamp (SFF) or sum trigger (SF4)."""
    c = list(c)
    x = 0
    raised = [0] * len(c)
    for op in ops:
        if op == 0:
            x += 1
            b = min(a + x for a in A)
            m = min(c)
            if m < b:
                for i in range(len(c)):
                    if c[i] == m:
                        c[i] += 1
                        raised[i] += 1
        else:
            x -= 1
            for i in range(len(c)):
                if sum_mode:
                    if c[i] > A[i] + x + O[i]:
                        c[i] -= 1
                else:
                    c[i] = min(c[i], max(A[i] + x, O[i]))
    return c, raised


def step_map(bits, W):
    """Per-word map exactly as word_maps_k builds it: (S, l, u, p0, pW)."""
    l, u, s, v0, vW, p0, pW = -INF, INF, 0, 0, W, 0, 0
    for d in bits:
        if d:
            l = l + 1
            u = min(u + 1, W)
            if l > u:
                l = u
            s += 1
            v0, vW = min(v0 + 1, W), min(vW + 1, W)
        else:
            l, u = max(l - 1, 0), max(u - 1, 0)
            s -= 1
            p0 += v0 == 0
            pW += vW == 0
            v0, vW = max(v0 - 1, 0), max(vW - 1, 0)
    return s, max(l, -INF), min(u, INF), p0, pW


def apply(f, v):
    s, l, u, _, _ = f
    return min(max(v + s, l), u)


def push(f, v):
    _, _, _, p0, pW = f
    return pW + max(p0 - pW - v, 0)


def cat(f, g, W):
    """rowmap_cat: f followed by g on [0, W]."""
    s1, l1, u1, p01, pW1 = f
    s2, l2, u2, _, _ = g
    L = max(l1 + s2, l2)
    U = min(max(u1 + s2, l2), u2)
    if L > U:
        L = U
    return (s1 + s2, max(L, -INF), min(U, INF), p01 + push(g, apply(f, 0)), pW1 + push(g, apply(f, W)))


def random_run(rng, sum_mode):
    d = rng.randint(1, 4)
    A = [rng.randint(20, 60) for _ in range(d)]
    A0 = min(A)
    if sum_mode:
        O = [rng.randint(0, 12) for _ in range(d)]
        Wd = [a - A0 + o for a, o in zip(A, O)]
    else:
        O = [rng.randint(0, a) for a in A]  # the key's own slot dominates
        Wd = [a - A0 for a in A]
    c = [A0 + rng.randint(0, w) for w in Wd]
    if not sum_mode:
        c[A.index(A0)] = A0  # SFF steady regime: the min sits at the own count
    n = rng.randint(1, 200)
    ops, cnt = [], rng.randint(0, 10)
    for _ in range(n):
        if cnt > 0 and rng.random() < rng.choice([0.2, 0.45, 0.49]):
            ops.append(1)
            cnt -= 1
        else:
            ops.append(0)
            cnt += 1
    if not sum_mode:  # keep the own slot dominant all run long, as the engine checks
        x, xmin = 0, 0
        for op in ops:
            x += -1 if op else 1
            xmin = min(xmin, x)
        O = [min(o, a + xmin) for o, a in zip(O, A)]
        if any(o < 0 for o in O):
            return None
    return A, O, c, ops, Wd


@pytest.mark.parametrize("sum_mode", [False, True])
def test_reflected_walk_pieces_match_replay(sum_mode):
    rng = random.Random(17 + sum_mode)
    checked = 0
    while checked < 3000:
        case = random_run(rng, sum_mode)
        if case is None:
            continue
        A, O, c, ops, Wd = case
        want_c, want_raised = replay(c, A, O, ops, sum_mode)
        A0 = min(A)
        x = sum(-1 if op else 1 for op in ops)
        # pieces of random lengths, composed with cat, then applied once
        cut = sorted(rng.sample(range(1, len(ops)), min(len(ops) - 1, rng.randint(0, 6))))
        bounds = [0] + cut + [len(ops)]
        for i, W in enumerate(Wd):
            f = None
            for a, b in zip(bounds[:-1], bounds[1:]):
                g = step_map(ops[a:b], W)
                f = g if f is None else cat(f, g, W)
            v = c[i] - A0
            assert apply(f, v) + A0 + x == want_c[i]
            assert push(f, v) == want_raised[i]
        checked += 1
