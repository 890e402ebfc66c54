"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
launch count, total and mean device time, and share of all qmpm kernel time.

    python profiles/summarize_launches.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if k.startswith(("qmpm", "qmpm::"))}
    allq = sum(ours.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        print(f"{k:40s} {cnt[k]:8d} {v:10.3f} {v / cnt[k]:9.3f} {100 * v / allq:5.1f}%")
    other = sum(v for k, v in tot.items() if k not in ours)
    print(f"(non-qmpm kernels in the process: {sum(c for k, c in cnt.items() if k not in ours)} launches, {other:.1f} ms: "
          "scene generation and torch setup)")


if __name__ == "__main__":
    main(sys.argv[1])
