"""Summarise an ncu report: SOL / occupancy / scheduler metrics and a
per-source-region breakdown of stall samples and executed instructions."""
import csv, subprocess, sys, io, json

rep = sys.argv[1]
ncand = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
regions = json.loads(sys.argv[3]) if len(sys.argv) > 3 else None

def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
hdr = det[0]
want = {"Duration", "Elapsed Cycles", "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate",
        "L2 Hit Rate", "DRAM Throughput", "Memory Throughput", "Eligible Warps Per Scheduler",
        "Avg. Active Threads Per Warp", "Compute (SM) Throughput"}
out = {}
for row in det[1:]:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        out[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'
for k, v in out.items():
    print(f"{k:40s} {v}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
rh = raw[0]
vals = dict(zip(rh, raw[2])) if len(raw) > 2 else {}
for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
    if m in vals:
        print(f"{m:40s} {vals[m]} {raw[1][rh.index(m)]}")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda,sass"]))))
cur = None; ph = {}; idx_s = idx_i = None
for r in src:
    if not r: continue
    if r[0] == "File Path": cur = r[1]; continue
    if r[0] == "Line No":
        idx_s = r.index("Warp Stall Sampling (All Samples)"); idx_i = r.index("Instructions Executed"); continue
    if not r[0].isdigit(): continue
    try: s = int(r[idx_s] or 0); i = int(r[idx_i] or 0)
    except Exception: continue
    key = (cur.split("/")[-1], int(r[0]), r[1][:80])
    a = ph.setdefault(key, [0, 0]); a[0] += s; a[1] += i
ts = sum(v[0] for v in ph.values()) or 1; ti = sum(v[1] for v in ph.values()) or 1
print(f"instructions/candidate {ti / ncand:.0f}")
for k, v in sorted(ph.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{k[0][:10]:10s}:{k[1]:<5d} s={100*v[0]/ts:5.1f}% i={100*v[1]/ti:5.1f}% {k[2]}")
if regions:  # {"name": [file_suffix, first_line, last_line], ...}
    print("per region (stall samples / instructions):")
    for name, (fs, lo, hi) in regions.items():
        s = sum(v[0] for k, v in ph.items() if k[0].startswith(fs) and lo <= k[1] <= hi)
        i = sum(v[1] for k, v in ph.items() if k[0].startswith(fs) and lo <= k[1] <= hi)
        print(f"  {name:24s} s={100*s/ts:5.1f}% i={100*i/ti:5.1f}% ({i / ncand:.0f} inst/candidate)")
