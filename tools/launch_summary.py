"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/launch_summary.py profiles/launches_r1e_candle.csv [--steps K]

--steps K divides the totals by K (per-step figures for a K-step capture).
"""
import collections
import csv
import re
import sys


def main(path, steps=1):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h, data = rows[0], rows[1:]
    ki, vi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    tot, cnt = collections.Counter(), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in data:
        if r[ni] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(anonymous namespace\)::|<?unnamed>::", "", r[ki])
        m = re.match(r"(?:void )?(?:[A-Za-z_0-9]+::)*([A-Za-z_0-9]+)(<[^(]*>)?", name)
        key = (m.group(1) + (m.group(2) or "")) if m else name[:60]
        us = float(r[vi].replace(",", "")) * (scale.get(r[ui], 1e-3) if ui is not None else 1e-3)
        tot[key] += us
        cnt[key] += 1
    T = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {T:.1f} us total (ncu: serialised, cold-cache)"
          + (f"; per step: {sum(cnt.values()) / steps:.0f} launches, {T / steps:.1f} us" if steps > 1 else ""))
    print(f"{'share':>6} {'n':>5} {'avg us':>9}  kernel")
    for k, v in tot.most_common():
        print(f"{100 * v / T:5.1f}% {cnt[k]:5d} {v / cnt[k]:9.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1)
