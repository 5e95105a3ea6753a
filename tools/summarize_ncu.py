"""Summarise ncu outputs into profiles/ (development tool).

  python tools/summarize_ncu.py <round-tag> <launches.csv> <report.ncu-rep> [<report2> ...]

Writes profiles/<tag>_launches.md (per-kernel share of device time in the bench's launch
list), profiles/<tag>_<report>.md (key metrics of each full capture) and
profiles/ncu_traffic.json (dram read+write bytes per launch of the dominant kernel, which
bench.py reports as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_active.avg", "sm__cycles_active.max", "gpc__cycles_elapsed.max", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def launches(path, tag):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        per[name][0] += 1
        per[name][1] += v
    tot = sum(v[1] for v in per.values()) or 1.0
    out = ["# %s -- ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-layers`" % tag, "",
           "Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum --clock-control none`):",
           "compare SHARES, not absolutes.  The list covers the whole process: layer synthesis (torch",
           "RNG/elementwise kernels) and packing (`pack_*`, one-time per layer) precede the timed region;",
           "a decode step launches only LUT-GEMV kernels -- `gemv_cluster_fused_kernel` (q/k/v fused),",
           "`gemv_cluster_ring_kernel` (o_proj, gate/up concatenated), `lut_stream_kernel` (down_proj, gate/up",
           "fused where the bit widths differ) -- plus the e2e leg's `copy_kernel`.", "",
           "| kernel | launches | total us | share of whole process |", "|---|---|---|---|"]
    for name, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        out.append("| `%s` | %d | %.1f | %.1f%% |" % (name, n, us, 100 * us / tot))
    with open(os.path.join(PROF, "%s_launches.md" % tag), "w") as f:
        f.write("\n".join(out) + "\n")
    return per


def report(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    name = os.path.basename(path).replace(".ncu-rep", "")
    out = ["# %s -- `ncu --set full` of `%s`" % (tag, name), ""]
    metrics = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        metrics.append(d)
        kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append("## %s" % kname.split("(")[0])
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        for k, (v, u) in d.items():
            out.append("| %s | %s | %s |" % (k, v, u))
        out.append("")
    with open(os.path.join(PROF, "%s_%s.md" % (tag, name)), "w") as f:
        f.write("\n".join(out) + "\n")
    return metrics


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(u, 1)


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(sys.argv[2], tag)
    # dram traffic per launch of every captured kernel, keyed by kernel id (bench.py's
    # roofline.traffic reads the dominant kernel's entry)
    ids = {"lut_stream_kernel": 8, "gemv_cluster_ring_kernel": 3, "gemv_cluster_fused_kernel": 10,
           "lut_program_kernel": 9}
    per_kernel = defaultdict(list)
    for rep in sys.argv[3:]:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        report(rep, tag)
        for vals in rows[2:]:
            kname = vals[hdr.index("Kernel Name")]
            kid = next((v for k, v in ids.items() if k in kname), None)
            if kid is None or "dram__bytes_read.sum" not in hdr:
                continue
            if "70b" in os.path.basename(rep):   # a per-layer shape, not a launch of the step
                kid = "%s_llama70b" % kid
            ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            t = to_bytes(vals[ir], units[ir]) + to_bytes(vals[iw], units[iw])
            per_kernel[str(kid)].append(t)
    out = {"round": tag, "kernels": {k: sum(v) / len(v) for k, v in per_kernel.items()},
           "per_launch_bytes": dict(per_kernel),
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the full captures (tools/evidence.sh); "
                   "the first launches of each kernel in a decode step: kernel 10 = q/k/v fused, kernel 3 = o_proj "
                   "and gate/up concatenated, kernel 8 = down_proj (and gate/up fused in blocks 20-31)"}
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("ok", tag, out["kernels"])
