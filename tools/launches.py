"""Summarise an ncu launch list (gpu__time_duration per launch): per-kernel
count / total / mean, restricted to the engine's kernels (rsvdb::) or all."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def main():
    path = sys.argv[1]
    only = len(sys.argv) > 2 and sys.argv[2] == "engine"
    agg = collections.OrderedDict()
    for d in load(path):
        name = d["Kernel Name"]
        if only and "rsvdb" not in name:
            continue
        v = float(d["Metric Value"])
        unit = d["Metric Unit"]
        v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        short = name.split("(")[0][:60] + ("<" + d["Grid Size"] + ">" if "pass_kernel" in name else "")
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:5d} {t:10.1f} us {t / c:9.2f} us/launch {100 * t / tot:5.1f}%  {k}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
