"""Instructions executed and stall samples of an ncu report summed over SASS
address ranges (offsets from the kernel start): python tools/sass_ranges.py
rep.csv name:start:end ... where rep.csv is `ncu -i rep --page source --csv
--print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, sass, seen = None, [], set()
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and len(r) > 2 and r[2].startswith("0x") and r[2] not in seen:
        seen.add(r[2])
        sass.append((int(r[2], 16), r[3].strip(), int(r[4] or 0), int(r[7] or 0)))
sass.sort()
base = sass[0][0]
ti = sum(s[3] for s in sass) or 1
ts = sum(s[2] for s in sass) or 1
print(f"total: {ti:.4g} warp-instructions, {ts} stall samples")
for spec in sys.argv[2:]:
    name, a, b = spec.split(":")
    a, b = int(a, 16), int(b, 16)
    sel = [s for s in sass if a <= s[0] - base < b]
    i = sum(s[3] for s in sel)
    st = sum(s[2] for s in sel)
    print(f"{name:>10}: instr {i / ti * 100:5.1f}%  stalls {st / ts * 100:5.1f}%")
