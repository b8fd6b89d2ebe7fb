import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsfsketch_cuda.so")


def fixture_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_fixture(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def load_hashing():
    with open(os.path.join(GOLDEN, "hashing.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    orc.lib()
    return orc


BASELINES = os.path.join(GOLDEN, "baselines")


def baseline_fixture_names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(BASELINES, prefix + "*.npz")))


def load_baseline_fixture(name):
    with np.load(os.path.join(BASELINES, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def parallel_engine_only():
    """Tiny and medium batches normally take the one-thread / warp / block
    engines (sfk_small_batch_ops, sfk_warp_batch_ops, sfk_block_batch_ops);
    parity tests turn those off so the parallel pipeline sees them too."""
    from paper_1701_04148_b200 import _lib

    L = _lib.lib()
    prev = L.sfk_small_batch_ops(0)
    prev_w = L.sfk_warp_batch_ops(0)
    prev_b = L.sfk_block_batch_ops(0)
    try:
        yield
    finally:
        L.sfk_small_batch_ops(prev)
        L.sfk_warp_batch_ops(prev_w)
        L.sfk_block_batch_ops(prev_b)
