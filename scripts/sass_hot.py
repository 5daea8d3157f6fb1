"""Per-instruction view of an ncu --set full capture (--import-source on): SASS offset, warp
instructions executed, average active threads, stall samples, instruction text -- and totals per
offset range.  Development aid for reading where the trace kernel's issue slots and stalls go.

    python scripts/sass_hot.py <capture.ncu-rep> [lo:hi:name ...]   (offsets in hex, kernel-relative)
"""
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rr) if r and r[0] == "Address")
    h = rr[hi]
    res = [dict(zip(h, r)) for r in rr[hi + 1:] if len(r) == len(h)]
    base = int(res[0]["Address"], 16)
    for d in res:
        d["off"] = int(d["Address"], 16) - base
    return res


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


def main():
    res = rows(sys.argv[1])
    tw = sum(f(d["Instructions Executed"]) for d in res)
    ts = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in res)
    ranges = [a.split(":") for a in sys.argv[2:]]
    if not ranges:
        for d in res:
            w = f(d["Instructions Executed"])
            print("%05x %12.0f %5.1f %6.0f  %s" % (d["off"], w, f(d["Avg. Threads Executed"]),
                                                  f(d["Warp Stall Sampling (All Samples)"]), d["Source"].strip()))
        return
    print("total warp inst %.4g, stall samples %.4g" % (tw, ts))
    for lo, hi, name in ranges:
        lo, hi = int(lo, 16), int(hi, 16)
        sel = [d for d in res if lo <= d["off"] < hi]
        w = sum(f(d["Instructions Executed"]) for d in sel)
        t = sum(f(d["Thread Instructions Executed"]) for d in sel)
        s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in sel)
        print("%-24s warp inst %5.1f %%  lanes %4.1f  stalls %5.1f %%" % (name, 100 * w / tw, t / max(w, 1), 100 * s / ts))


if __name__ == "__main__":
    main()
