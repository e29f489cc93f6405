"""Summarise an ncu report's source page: hottest CUDA source lines by warp-stall samples.

    python tools/ncu_hotlines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, lines = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name", "Kernel Name") and len(r) >= 8:
        try:
            samples = int(r[4])
            execd = int(r[7])
        except ValueError:
            continue
        lines.append((samples, execd, cur, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in lines)
print(f"total samples {tot}")
for s, e, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100.0 * s / max(tot, 1):5.1f}% {s:8d} {e:11d} {f}:{ln:5s} {src}")
