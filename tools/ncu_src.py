"""Summarise an ncu --page source csv (SASS): per-instruction stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
tot = sum(int(r[iS]) for r in data); ins = sum(int(r[iE]) for r in data)
print("samples", tot, "warp-instructions", ins)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {int(r[iS]):6d} {int(r[iE]):8d}  {r[1][:90]}")
