"""Refresh profiles/trace_traffic.json and profiles/trace_profile.json (read by bench.py for the
roofline's `traffic` and L1 second ceiling) from one ncu --set full capture of k_trace_stereo.

    python scripts/update_trace_profile.py <tag> <capture.ncu-rep>
"""
import csv
import io
import json
import subprocess
import sys

tag, rep = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
u = dict(zip(h, units))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1.0, "msecond": 1.0, "usecond": 1e-3,
         "nsecond": 1e-6, "%": 1.0, "": 1.0}


def f(k):
    return float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)


src = (f"profiles/{tag}.md (ncu --set full, {d['Kernel Name'][:40]}, C4 1080p stereo d4, one launch, "
       "L2 cold after the flush)")
traffic = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
json.dump({"C4/x1": traffic,
           "_note": "dram__bytes_read.sum + dram__bytes_write.sum of one k_trace_stereo launch, " + src},
          open("profiles/trace_traffic.json", "w"), indent=1)
sectors = f("l1tex__t_sectors.sum") if "l1tex__t_sectors.sum" in d else f("SM_B.TriageCompute.l1tex__t_sectors.sum")
wf = f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")
prof = {"C4/x1": {"l1tex_t_bytes": sectors * 32.0, "l1tex_t_sectors": sectors,
                  "l1tex_data_pipe_lsu_wavefronts_pct_peak": wf, "l1tex_throughput_pct_peak": wf,
                  "gpu_time_ms": f("gpu__time_duration.sum"), "source": src},
        "_note": "l1tex_t_bytes = l1tex__t_sectors.sum x 32 B (every L1 tag lookup of the launch, hits and misses); "
                 "the L1 data pipe (LSU wavefronts) runs at the listed % of its peak: incoherent 128-bit loads cost "
                 "a wavefront per distinct line"}
json.dump(prof, open("profiles/trace_profile.json", "w"), indent=1)
print(json.dumps({"traffic": traffic, **prof["C4/x1"]}, indent=1))
