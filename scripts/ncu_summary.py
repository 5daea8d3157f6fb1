"""Summarise an ncu capture (--set full) and an ncu launch list into profiles/<tag>.{json,md}.

usage: python scripts/ncu_summary.py <tag> <full.ncu-rep> [launches.csv] [bench.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
    "smsp__sass_branch_targets_threads_divergent.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__inst_executed.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, name in enumerate(h):
            if name in KEYS or name in ("Kernel Name", "ID"):
                d[name] = r[i] + (f" {units[i]}" if units[i] and name not in ("Kernel Name", "ID") else "")
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ks = []
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        ks.append((d["Kernel Name"], float(d["Metric Value"])))
    return ks


def main():
    tag, rep = sys.argv[1], sys.argv[2]
    lpath = sys.argv[3] if len(sys.argv) > 3 else None
    bpath = sys.argv[4] if len(sys.argv) > 4 else None
    os.makedirs("profiles", exist_ok=True)
    summ = {"tag": tag, "capture": raw(rep)}
    md = [f"# ncu summary {tag}", "", "## --set full capture (top kernel)", ""]
    for k in summ["capture"]:
        md.append(f"### {k.get('Kernel Name', '?')[:100]}")
        for key in KEYS:
            if key in k:
                md.append(f"- `{key}` = {k[key]}")
        md.append("")
    if lpath:
        ks = launches(lpath)
        summ["launches"] = ks
        md += ["## launch list (gpu__time_duration.sum, --clock-control none, cold & serialised)", "",
               "| # | kernel | ns |", "|---|---|---|"]
        for i, (n, t) in enumerate(ks):
            md.append(f"| {i} | `{n[:80]}` | {t:.0f} |")
        trace = [t for n, t in ks if "k_trace_stereo<0" in n or "k_trace_stereo<false" in n]
        other = [t for n, t in ks if ("k_unpack" in n)]
        if trace:
            md += ["", f"trace kernel (uninstrumented) launches: {len(trace)}, mean {sum(trace) / len(trace) / 1e3:.3f} us"]
            summ["trace_kernel_mean_ns"] = sum(trace) / len(trace)
    if bpath:
        try:
            b = json.loads(open(bpath).read().strip().splitlines()[-1])
            summ["bench"] = b
            md += ["", "## bench line", "", "```", json.dumps(b, indent=1)[:4000], "```"]
        except Exception as e:  # noqa: BLE001
            md += ["", f"(bench parse failed: {e})"]
    json.dump(summ, open(f"profiles/{tag}.json", "w"), indent=1)
    open(f"profiles/{tag}.md", "w").write("\n".join(md) + "\n")
    print("\n".join(md[:60]))


if __name__ == "__main__":
    main()
