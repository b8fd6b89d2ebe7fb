"""CPU-only checks of the product's host side: the C-ABI library loads and
exports every symbol include/sfsketch_cuda.h declares (no compute calls), the
host hash family matches the reference goldens, parameter validation and the
export-format parser behave like the reference's."""

import os
import re
import struct

import numpy as np
import pytest

from conftest import ROOT, load_fixture, load_hashing

from paper_1701_04148_b200 import _lib, errors, hashing
from paper_1701_04148_b200.params import SketchParams


def header_functions():
    src = open(os.path.join(ROOT, "include", "sfsketch_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sfk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    L = _lib.load_library()
    names = header_functions()
    assert set(names) == set(_lib.EXPORTS)
    for name in names:
        assert hasattr(L, name), name
    assert L.sfk_abi_version() == 1


def test_nm_shows_extern_c_symbols():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sfk_\w+)", out))
    assert set(header_functions()) <= exported


def test_host_hash_family_matches_reference_goldens():
    h = load_hashing()
    for k, want in h["finalize"].items():
        assert hashing.finalize64(int(k)) == int(want)
    ins = np.array([int(x) for x in h["mix_batch_in"]], dtype=np.uint64)
    assert [str(int(v)) for v in hashing.finalize64_array(ins)] == h["mix_batch_out"]
    for key, want in h["seeds"].items():
        m, d = (int(x) for x in key.split(":"))
        assert [str(s) for s in hashing.derive_seeds(m, d).per_array_seeds] == want
    for s, want in h["key_from_string"].items():
        assert hashing.key_from_string(s) == int(want)
    fam = hashing.derive_seeds(6, 4)
    for k, i, r, want in h["bucket"]:
        assert hashing.bucket_hash(fam, i, int(k), r) == want
    for k, i, z, want in h["slot"]:
        assert hashing.slot_hash(fam, i, int(k), z) == want
    assert hashing.seed_for_index(0, 0) == 0xE220A8397B1DCDAF
    assert hashing.key_from_string("apple") == 0xBA8E799DCEB3BCB1


def test_params_validation():
    p = SketchParams(d=4, w=16384, z=4)
    assert p.w_prime == 65536
    for bad in [dict(d=0, w=4), dict(d=1, w=0), dict(d=1, w=4, z=0), dict(d=2, w=8, w_prime=4),
                dict(d=1, w=4, master_seed=-1), dict(d=1, w=4, epsilon=0.1)]:
        with pytest.raises(errors.ConfigurationError):
            SketchParams(**bad)
    q = SketchParams.from_error_bounds(0.01, 0.05)
    assert (q.d, q.w) == (3, 272)
    with pytest.raises(errors.ConfigurationError):
        SketchParams(d=4, w=272, epsilon=0.01, delta=0.05)


def test_import_slim_parser_errors_and_roundtrip():
    from paper_1701_04148_b200.serialize import HEADER, import_slim

    fx = load_fixture("sff_u32_medium")
    payload = fx["export"].tobytes()
    col = import_slim(payload)
    assert col.export() == payload
    np.testing.assert_array_equal(col.counters, fx["slim"])
    assert col.insertions_seen == int(fx["seen"])
    with pytest.raises(ValueError):
        col.counters[0, 0] = 1
    with pytest.raises(errors.BadMagicError):
        import_slim(b"XXXX" + payload[4:])
    with pytest.raises(errors.PayloadLengthError):
        import_slim(payload[:20])
    with pytest.raises(errors.PayloadLengthError):
        import_slim(payload[:-1])
    with pytest.raises(errors.PayloadLengthError):
        import_slim(payload + b"\0")
    magic, ver, code, res, d, w, ms, seen = HEADER.unpack_from(payload)
    with pytest.raises(errors.UnsupportedVersionError):
        import_slim(HEADER.pack(magic, 2, code, res, d, w, ms, seen) + payload[32:])
    with pytest.raises(errors.UnknownVariantCodeError):
        import_slim(HEADER.pack(magic, ver, 5, res, d, w, ms, seen) + payload[32:])
    with pytest.raises(errors.ExportFormatError):
        import_slim(HEADER.pack(magic, ver, code, 1, d, w, ms, seen) + payload[32:])


def test_empty_sff_export_golden_bytes():
    # tests/test_serialize.py:30-43 of the reference: empty SFF d=2, w=4
    from paper_1701_04148_b200.serialize import _pack

    want = struct.pack("<4sBBHIIQQ", b"SFSK", 1, 6, 0, 2, 4, 0, 0) + bytes(32)
    assert _pack(6, 2, 4, 0, 0, bytes(32)) == want
    assert len(want) == 64
