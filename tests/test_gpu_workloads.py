"""The reference's synthetic streams generated on the GPU
(workloads.generate: numpy's PCG64 stream evaluated in parallel on the
device, Zipf ranks by the same CDF search, the interleaved-deletion walk in a
device thread) against what the reference's generate produced for the same
specs (tests/golden/make_golden_workloads.py). Plus the raw PCG64 draws
against numpy at arbitrary stream offsets."""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

FX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "streams", "workloads.npz")


def load():
    with np.load(FX) as z:
        d = {k: z[k] for k in z.files}
    return d, json.loads(d["meta"].tobytes().decode())


@pytest.mark.parametrize("name", sorted(load()[1]))
def test_generate_matches_reference(oracle, name):
    d, meta = load()
    wl = W.generate(W.WorkloadSpec(**meta[name]))
    np.testing.assert_array_equal(wl.ops.cpu().numpy(), d[name + "_ops"])
    np.testing.assert_array_equal(wl.ranks.cpu().numpy(), d[name + "_ranks"])
    np.testing.assert_array_equal(wl.keys.cpu().numpy(), oracle.mix_batch(d[name + "_ranks"].astype(np.uint64)))


@pytest.mark.parametrize("seed,offset,n", [(0, 0, 1), (7, 0, 100_000), (2017, 123_456_789, 5000),
                                           (2**64 - 1, 10**12, 300)])
def test_pcg64_draws_equal_numpy(seed, offset, n):
    g = np.random.Generator(np.random.PCG64(seed))
    st = g.bit_generator.state["state"]
    m64 = (1 << 64) - 1
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().sfk_pcg64_draws(st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64,
                                          offset, n, None, 0, None, out.data_ptr(), _lib.stream_ptr()), "draws")
    g.bit_generator.advance(offset)
    np.testing.assert_array_equal(out.cpu().numpy(), g.random(n))


@pytest.mark.parametrize("seed,v,n,skip", [(6, 777, 30_000, 0), (1, 1, 100, 0), (3, 2**31 + 1, 50_000, 0),
                                           (4, 2**32, 1000, 0), (5, 1_000_003, 200_000, 12345), (8, 3, 1, 0)])
def test_pcg64_bounded_equal_numpy(seed, v, n, skip):
    """Generator.integers(0, v, dtype=int64) from the device, including the
    stream position it leaves (checked through the next random() draws)."""
    g = np.random.Generator(np.random.PCG64(seed))
    st = g.bit_generator.state["state"]
    m64 = (1 << 64) - 1
    L = _lib.lib()
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    ws = torch.empty(int(L.sfk_pcg64_bounded_workspace_size(n, v)), dtype=torch.uint8, device="cuda")
    nxt = np.zeros(1, dtype=np.int64)
    _lib.check(L.sfk_pcg64_bounded(st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64, skip, n, v,
                                   out.data_ptr(), nxt.ctypes.data, ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
               "bounded")
    g.bit_generator.advance(skip)
    np.testing.assert_array_equal(out[:n].cpu().numpy(), g.integers(0, v, size=n, dtype=np.int64))
    h = np.random.Generator(np.random.PCG64(seed))
    h.bit_generator.advance(int(nxt[0]))
    np.testing.assert_array_equal(h.random(4), g.random(4))
