"""Sum an ncu --metrics gpu__time_duration.sum --csv launch list by kernel
(ms per kernel, share, launches). Usage: python tools/launch_sum.py launches.csv"""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum": continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    ms = v / 1e6 if u in ("nsecond", "ns") else v / 1e3 if u in ("usecond", "us") else v if u in ("msecond", "ms") else v / 1e6
    k = r[ki][:90]
    a = agg.setdefault(k, [0.0, 0]); a[0] += ms; a[1] += 1
tot = sum(a[0] for a in agg.values())
for k, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print("%9.3f ms %5.1f%% x%-4d %s" % (ms, 100 * ms / tot, c, k))
print("%9.3f ms total" % tot)
