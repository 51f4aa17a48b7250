"""Per-kernel share of an ncu launch list (`ncu --metrics gpu__time_duration.sum
--csv --log-file X`): launches, total ns and share of the summed device time.
ncu serialises launches and runs them cold-cache, so read shares, not times."""
import csv
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = name.replace("void ", "", 1)
    depth, out = 0, []
    for ch in name:  # drop the argument list, keep the template arguments
        if ch == "(" and depth == 0:
            break
        depth += ch == "<"
        depth -= ch == ">"
        out.append(ch)
    s = "".join(out)
    return s if len(s) <= 90 else s[:87] + "..."


def main(path: str, title: str = "") -> None:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0}.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(short(r["Kernel Name"]), [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    print(f"kernel, launches, total_ns, share  ({title})")
    for k, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k}, {cnt}, {ns:.0f}, {ns / tot * 100:.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
