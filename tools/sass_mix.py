"""Dynamic SASS opcode mix and stall samples of one kernel from an ncu report
(`ncu -i X --page source --csv --print-source sass`), per unit of work."""
import csv
import subprocess
import sys
from collections import Counter


def main(rep: str, units: float = 1.0) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    hdr = rows[0]
    isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stall = Counter(), Counter()
    for r in rows[1:]:
        op = r[isrc].strip().split()[0] if r[isrc].strip() else "?"
        if op.startswith("@"):
            op = r[isrc].strip().split()[1]
        op = op.split(".")[0]
        cnt[op] += float(r[iex] or 0)
        stall[op] += float(r[ist] or 0)
    tot, stot = sum(cnt.values()), sum(stall.values())
    print(f"{'opcode':10s} {'per unit':>12s} {'share':>7s} {'stall%':>7s}")
    for op, v in cnt.most_common(40):
        print(f"{op:10s} {v / units:12.1f} {v / tot * 100:6.2f}% {stall[op] / stot * 100:6.2f}%")
    print(f"{'total':10s} {tot / units:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
