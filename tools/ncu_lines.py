"""Per-CUDA-line stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.008
out = []
hdr = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        out.append((int(r[0]), int(r[4]), int(r[7]), r[1].strip()))
    except ValueError:
        pass
tot = sum(x[1] for x in out) or 1
ins = sum(x[2] for x in out)
print("samples", tot, "warp-instr", ins)
for ln, s, e, src in out:
    if s > tot * thr:
        print(f"{ln:4d} {s:7d} {100*s/tot:5.1f}% {e:10d}  {src[:85]}")
