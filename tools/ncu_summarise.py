"""Condense an ncu report into committed text evidence under profiles/.

    python tools/ncu_summarise.py REP.ncu-rep OUT_PREFIX [STEPS]

writes OUT_PREFIX_raw.csv    every metric of the captured launch(es)
                             (`ncu -i REP --page raw --csv`)
       OUT_PREFIX_lines.txt  per CUDA source line: share of warp-stall
                             samples and instructions per step (when the
                             report has SourceCounters and STEPS is given),
                             plus the stall-reason totals
"""
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    steps = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    raw = ncu(rep, "--page", "raw", "--csv")
    with open(out + "_raw.csv", "w") as fh:
        fh.write(raw)
    src = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    rows = list(csv.reader(io.StringIO(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hi:
        return
    hdr, data = rows[hi[0]], rows[hi[0] + 1:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0

    lines, totals = [], {}
    for r in data:
        if len(r) > iE and r[0].isdigit():
            lines.append((int(r[0]), r[1].strip()[:90], num(r[iS]), num(r[iE])))
        elif len(r) > iE and r[2].startswith("0x"):
            for i in stall:
                totals[hdr[i]] = totals.get(hdr[i], 0) + num(r[i])
    tot = sum(x[2] for x in lines) or 1
    ins = sum(x[3] for x in lines)
    with open(out + "_lines.txt", "w") as fh:
        fh.write(f"# {rep}\n# warp-stall samples {tot}, instructions {ins}"
                 + (f", steps {steps:.0f}, instructions/step {ins / steps:.1f}" if steps else "")
                 + "\n# stall reasons (share of samples):\n")
        st = sum(totals.values()) or 1
        for k, v in sorted(totals.items(), key=lambda x: -x[1])[:10]:
            fh.write(f"#   {k:28s} {100 * v / st:5.1f} %\n")
        fh.write("# line  samples%  instr/step  source\n")
        for ln, txt, s, e in sorted(lines, key=lambda x: -x[2])[:60]:
            per = f"{e / steps:8.2f}" if steps else f"{e:10d}"
            fh.write(f"{ln:6d} {100 * s / tot:7.2f}% {per}  {txt}\n")


if __name__ == "__main__":
    main()
