"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel device time of ONE pipeline step (the last complete step before
the end of the capture), with shares. Steps start at k_prepare.
    python tools/launch_summary.py launches.csv [out.csv]"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*$", "", name)
    for junk in ("wsb::<unnamed>::", "unnamed>::", "void "):
        name = name.replace(junk, "")
    return name.strip()


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "nsecond" or unit == "ns" else (v if unit in ("usecond", "us") else v * 1e3)
        rows.append((int(r["ID"]), short(r["Kernel Name"]), us))
    starts = [i for i, (_, k, _) in enumerate(rows) if k in ("k_prepare", "k_count<true>", "k_count<1>")]
    if len(starts) >= 2:
        a, b = starts[-2], starts[-1]
    else:
        a, b = (starts[0] if starts else 0), len(rows)
    step = rows[a:b]
    agg = OrderedDict()
    for _, k, us in step:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    out = ["kernel,launches,us,share"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k},{n},{t:.1f},{t / total:.3f}")
    out.append(f"TOTAL,{sum(n for n, _ in agg.values())},{total:.1f},1.000")
    text = "\n".join(out)
    print(text)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
