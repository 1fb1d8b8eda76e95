"""Per-CUDA-line warp-stall summary of an ncu report (needs -lineinfo builds):
    python scripts/ncu_lines.py REPORT.ncu-rep [first_line last_line] [top]
Prints the lines with the most stall samples and their top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10 ** 9)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, hdr = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        ln = int(r[0])
        if not (lo <= ln <= hi):
            continue
        samp = int(r[4]) if r[4].isdigit() else 0
        stalls = {hdr[i]: int(r[i] or 0) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]
                  and (r[i] or "0").isdigit()}
        res.append((samp, fname, ln, r[1].strip()[:70], sorted(stalls.items(), key=lambda x: -x[1])[:3], r[7]))
tot = sum(x[0] for x in res)
print("samples in range:", tot)
for samp, f, ln, src, st, ex in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{samp:7d} {100 * samp / max(tot, 1):5.1f}% {f}:{ln:5d} ex={ex:>9s} {src:70s} {' '.join(f'{k[6:]}={v}' for k, v in st)}")
