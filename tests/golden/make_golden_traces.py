"""Trace-format fixtures: crafted trace files and what the REFERENCE's
load_trace makes of them (build container only; imports /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_traces.py

Writes tests/golden/traces/<name>.trace and expected.json:
{name: {"ops": [...], "keys": [str...]} or {"error_line": n, "message": str}}.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from sfsketch.errors import TraceFormatError  # noqa: E402
from sfsketch.workloads import WorkloadSpec, generate, load_trace, write_trace  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traces")

CASES = {
    "basic": b"# comment\nI,42\nI,42\nD,42\n",
    "empty": b"",
    "blank_lines": b"\n\n  \nI,1\n\t\nD,1\n\n",
    "crlf": b"I,1\r\nI,2\r\n# c\r\nD,1\r\n",
    "lone_cr": b"I,1\rI,2\rD,1\r",
    "mixed_newlines": b"I,1\r\nI,2\rI,3\nD,3",
    "no_final_newline": b"I,18446744073709551615",
    "whitespace": b"  I , 7  \n\tD\t,\t7\x0b\n\x0cI,\x1c8\x1f\n",
    "signs_underscores": b"I,+5\nI,-0\nI,1_000_000\nI,007\nD,+1_0\n",
    "max_key": b"I,18446744073709551615\nD,18446744073709551615\n",
    "comment_after_ws": b"   # indented comment\nI,3\n#I,4\n",
    "unicode_ws": "I, 5\nI, 6　\n".encode("utf-8"),
    "unicode_digits": "I,١٢\n".encode("utf-8"),
    "bad_token": b"X,5\n",
    "bad_sep": b"I;5\n",
    "bad_key": b"I,notakey\n",
    "three_parts": b"I,5,6\n",
    "too_big": b"I,99999999999999999999999\n",
    "negative": b"I,1\nD,-5\n",
    "bad_after_comments": b"# header\nI,1\n\nD,oops\n",
    "bad_underscore": b"I,1__0\n",
    "trailing_underscore": b"I,10_\n",
    "empty_key": b"I,\n",
    "empty_token": b",5\n",
    "lowercase": b"i,5\n",
    "space_in_key": b"I,1 2\n",
    "bad_line_crlf": b"I,1\r\nI,2\r\nQ,3\r\n",
    "hex_key": b"I,0x10\n",
    "plus_only": b"I,+\n",
    "unicode_bad": "I,5\nI,é\n".encode("utf-8"),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    expected = {}
    spec = WorkloadSpec(kind="zipf", distinct_items=300, total_ops=20_000, seed=5, deletion_mode="interleaved",
                        delete_prob=0.3)
    wl = generate(spec)
    big = os.path.join(OUT, "roundtrip.trace")
    write_trace(big, wl.operations())
    for name, data in CASES.items():
        with open(os.path.join(OUT, name + ".trace"), "wb") as fh:
            fh.write(data)
    for name in sorted(list(CASES) + ["roundtrip"]):
        path = os.path.join(OUT, name + ".trace")
        try:
            ops, keys = load_trace(path)
            expected[name] = {"ops": [int(o) for o in ops], "keys": [str(int(k)) for k in keys]}
        except TraceFormatError as e:
            expected[name] = {"error_line": e.line_number, "message": str(e)}
    with open(os.path.join(OUT, "expected.json"), "w") as fh:
        json.dump(expected, fh, indent=1, sort_keys=True)
    print(json.dumps({k: (v.get("error_line") or len(v["ops"])) for k, v in expected.items()}))


if __name__ == "__main__":
    main()
