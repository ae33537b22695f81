"""Per-source-line executed warp-instructions and stall samples per planner
step, from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_steps.py src.csv steps [min_instr_per_step]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]); thr = float(sys.argv[3]) if len(sys.argv) > 3 else 2.0
hdr = None; f = None; out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        out.append((f, int(r[0]), int(r[4]), int(r[7]), r[1].strip()))
    except ValueError:
        pass
ts = sum(o[2] for o in out) or 1
ti = sum(o[3] for o in out)
print(f"instr/step {ti / steps:.1f}  samples {ts}")
for f, ln, s, e, src in out:
    if e / steps >= thr or s > 0.01 * ts:
        print(f"{f[:12]:12s}{ln:5d} {e / steps:7.1f} {100 * s / ts:5.1f}%  {src[:80]}")
