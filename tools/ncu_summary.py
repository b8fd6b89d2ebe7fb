"""Condense an ncu --set full report into the numbers the roofline cites:
duration, DRAM bytes (the `traffic` field), L2 sectors, shared-memory
wavefronts, issue/occupancy and the top warp-stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep > summary.txt
       python tools/ncu_summary.py --traffic report.ncu-rep name units unit_name"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second",
]

def summarize(rep):
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "?")[:120])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>22s} {u.get(k, '')}")
        stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")]
        vals = []
        for k, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
        print("  top stall reasons (warps stalled per issue-active cycle):")
        for v, k in sorted(vals, reverse=True)[:8]:
            print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:40s} {v:8.3f}")


def record_traffic(rep, name, units, unit_name, out="profiles/ncu_traffic.json"):
    """Store DRAM bytes per unit of `name` (from one --set full capture) for
    bench.py's roofline `traffic` field."""
    import json
    import os

    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(k):
        return float(d[k].replace(",", "")) * scale.get(u[k], 1)

    tot = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    db = json.load(open(out)) if os.path.exists(out) else {}
    db[name] = {"dram_bytes": tot, "units": units, "unit": unit_name, "bytes_per_unit": tot / units,
                "kernel": d.get("Kernel Name", "")[:160], "report": os.path.basename(rep)}
    json.dump(db, open(out, "w"), indent=1)


if __name__ == "__main__":
    if len(sys.argv) >= 5 and sys.argv[1] == "--traffic":
        # python tools/ncu_summary.py --traffic report.ncu-rep name units unit_name
        record_traffic(sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5] if len(sys.argv) > 5 else "unit")
    else:
        summarize(sys.argv[1])
