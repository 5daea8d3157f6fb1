"""SASS-derived ceiling of the trace kernel (VERDICT r1 "turn 60 % is unreachable into a measured
ceiling"): per-instruction execution counts from an ncu --set full capture (--import-source, source
page), classified by pipe, against the algorithmic flops of the same launch.

    python scripts/sass_mix.py <capture.ncu-rep> <bench.json> [--kernel regex] > profiles/<tag>_sass_mix.json

The decomposition (all measured, one launch):
    frac = issue_eff x simt_eff x mix_ceiling
      issue_eff   = warp instructions issued / (issue slots of the launch: 4 SMSP x 148 SM x cycles)
      simt_eff    = thread instructions / (32 x warp instructions)
      mix_ceiling = algorithmic flops per thread instruction / (peak flops per issued thread
                    instruction: 256 flop/clk/SM over 128 issued thread-instructions/clk/SM = 2)
mix_ceiling is the FP32 fraction this instruction stream would reach at 100 % issue and 32/32 lanes.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

FMA = {"FFMA", "FMUL", "FADD", "FFMA2", "FMUL2", "FADD2", "IMAD", "HFMA2", "HADD2", "HMUL2", "FHFMA"}
ALU = {"IADD3", "LOP3", "SHF", "PRMT", "FMNMX", "FMNMX3", "ISETP", "FSETP", "SEL", "FSEL", "PLOP3", "VIMNMX", "IMNMX",
       "LEA", "MOV", "VIADD", "IABS", "FLO", "POPC", "BREV", "P2R", "R2P", "ICMP", "FCHK", "IADD", "LEA.HI", "UISETP"}
LSU = {"LDG", "LDS", "STS", "LDL", "STL", "STG", "ATOMG", "RED", "LD", "ST", "ATOM", "ATOMS", "LDC", "SHFL"}
XU = {"MUFU", "I2F", "F2I", "F2F", "I2FP", "F2FP", "FRND"}
CTRL = {"BRA", "BSSY", "BSYNC", "BREAK", "EXIT", "RET", "CALL", "WARPSYNC", "BAR", "NOP", "YIELD", "VOTE", "VOTEU",
        "BMOV", "NANOSLEEP", "MATCH", "REDUX", "ELECT", "ENDCOLLECTIVE"}


def pipe_of(op):
    base = op.split(".")[0]
    if base.startswith("U") and base not in ("UISETP",):   # uniform datapath
        return "uniform"
    for name, s in (("fma", FMA), ("alu", ALU), ("lsu", LSU), ("xu", XU), ("ctrl", CTRL)):
        if base in s:
            return name
    return "other"


def source_page(rep, kernel):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    res = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        res.append(d)
    return res


def raw_metric(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    i = rows[0].index(name)
    return float(rows[2][i].replace(",", ""))


def main():
    rep, bench = sys.argv[1], sys.argv[2]
    kernel = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    rows = source_page(rep, kernel)
    warp = defaultdict(float)
    thr = defaultdict(float)
    ops = defaultdict(float)
    for d in rows:
        src = d["Source"].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)", src)
        if not m:
            continue
        op = m.group(2)
        w = float(d["Instructions Executed"] or 0)
        t = float(d["Thread Instructions Executed"] or 0)
        p = pipe_of(op)
        warp[p] += w
        thr[p] += t
        ops[op.split(".")[0]] += t
    W = sum(warp.values())
    T = sum(thr.values())
    b = json.loads(open(bench).read().strip().splitlines()[-1])
    flops = b["roofline"]["algorithmic_flops_per_launch"]
    cycles = raw_metric(rep, "sm__cycles_elapsed.avg")
    issue_eff = W / (4 * 148 * cycles)
    simt = T / (32 * W)
    mix = (flops / T) / 2.0
    out = {
        "capture": rep, "warp_instructions": W, "thread_instructions": T, "sm_cycles": cycles,
        "algorithmic_flops": flops,
        "by_pipe_warp_inst": dict(sorted(warp.items(), key=lambda x: -x[1])),
        "by_pipe_thread_inst_share": {k: v / T for k, v in sorted(thr.items(), key=lambda x: -x[1])},
        "top_opcodes_thread_inst_share": {k: v / T for k, v in sorted(ops.items(), key=lambda x: -x[1])[:25]},
        "issue_eff": issue_eff, "simt_eff": simt, "mix_ceiling": mix,
        "frac_model": issue_eff * simt * mix,
        "frac_bench": b["roofline"]["frac"],
        "note": "frac = issue_eff x simt_eff x mix_ceiling; mix_ceiling = the FP32 fraction at 100 % issue "
                "and 32/32 lanes (algorithmic flops per thread instruction / 2)",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
