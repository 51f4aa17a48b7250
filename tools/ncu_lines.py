"""Per-source-line warp-stall samples and excess shared wavefronts from an ncu
report (`--import-source on`): python tools/ncu_lines.py rep.ncu-rep [top]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, f, hdr = [], None, None
for r in csv.reader(out):
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:  # a CUDA line (SASS rows have no line number)
        try:
            s = int(r[4] or 0)
        except ValueError:
            continue
        exc = r[hdr.index("L1 Wavefronts Shared Excessive")] if "L1 Wavefronts Shared Excessive" in hdr else ""
        rows.append((s, f, r[0], r[1].strip()[:80], exc))
tot = sum(r[0] for r in rows) or 1
print(f"total stall samples {tot}")
for s, fn, ln, src, exc in sorted(rows, reverse=True)[:top]:
    print(f"{s / tot * 100:5.1f}%  {fn}:{ln}  excess_smem_wf={exc}  | {src}")
