"""SASS census of the hot kernels (no GPU needed): per kernel, counts of the
sm_100 instructions that show which hardware paths they use (DSMEM st.async,
mbarrier SYNCS ops, cluster MAPA, 256-bit stores, shared loads, ...).
Counts match by prefix, so STG includes STG.E.EF.ENL2.256 and SYNCS its
ARRIVE/PHASECHK forms.
Usage: python tools/sass_census.py > profiles/r02/sass_census.txt"""
import re
import subprocess
import sys
from collections import Counter

OBJS = ["paper_1701_04148_b200/_build/sfk_query.o", "paper_1701_04148_b200/_build/sfk_sf.o"]
KERNELS = [r"min_query_cwILi4EtLi16ELi16ELi4ELb1ELb0E", r"poll_engine_kILi4ELi2E", r"segscan_apply_kILi4ELb1ELi2ELb1E",
           r"runs_build_kILi4E", r"cm_atomic_kILi4E"]
OPS = ["STAS", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "SYNCS", "MAPA", "UBLKCP", "UTMALDG", "LDS", "LDS.U16", "STG.E.EF.ENL2.256", "LDG.E.ENL2.256", "STG",
       "LDG", "REDG", "RED", "ATOMG", "ATOMS", "VIMNMX3", "VIMNMX", "IMAD", "NANOSLEEP", "BAR.SYNC", "ELECT", "UCGABAR_ARV", "UCGABAR_WAIT", "CCTL"]


def census(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)[1:]
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if not any(re.search(k, name) for k in KERNELS):
            continue
        mnem = Counter()
        for line in f.split("\n"):
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                mnem[m.group(1)] += 1
        print(f"== {name}  ({sum(mnem.values())} SASS instructions)")
        for op in OPS:
            n = sum(c for k, c in mnem.items() if k == op or k.startswith(op + "."))
            if n:
                print(f"   {op:22s} {n}")


for o in (sys.argv[1:] or OBJS):
    census(o)
