"""Per-kernel summary of an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(tools/one_step.py runs `steps` factorizations): launches per factorization,
mean time, and DRAM read + write bytes per launch.

  python tools/ncu_traffic.py gpurun_out/r02_launches_C5.csv [steps]
"""
import collections
import csv
import glob
import os
import re
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def engine_kernels():
    """__global__ function names of the engine (paper_2402_17794_b200/csrc)."""
    names = set()
    skip = {"void", "__launch_bounds__", "__global__", "__noinline__", "__forceinline__"}
    for f in glob.glob(os.path.join(HERE, "paper_2402_17794_b200", "csrc", "*.cu*")):
        src = open(f).read()
        for m in re.finditer(r"__global__", src):
            for ident in re.findall(r"(\w+)\s*\(", src[m.end():m.end() + 300]):
                if ident not in skip and not ident.isupper() and ident != "CW":
                    names.add(ident)
                    break
    return names


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    ix = {k: i for i, k in enumerate(hdr)}
    per = collections.OrderedDict()  # (launch id) -> dict
    for r in rows:
        if r[0] == "ID" or len(r) != len(hdr):
            continue
        d = per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
        try:
            v = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        unit = r[ix["Metric Unit"]]
        name = r[ix["Metric Name"]]
        if name == "gpu__time_duration.sum":
            v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
            d["us"] = v
        elif name.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[name] = v * scale
    ours = engine_kernels()
    agg = collections.OrderedDict()
    for d in per.values():
        short = d["name"].replace("rsvdb::", "").replace("<unnamed>::", "").replace("void ", "")
        short = short.split("(")[0].strip()
        base = re.sub(r"<.*", "", short).split("::")[-1]
        if base not in ours:
            continue
        if base in ("pass_kernel", "fused_pass_kernel"):
            short = base + short[len(base):].split(">")[0][:26] + ("> grid " + d["grid"])
        if "us" not in d:  # not profiled (e.g. a kernel that waits on the host)
            continue
        a = agg.setdefault(short, {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["us"] += d.get("us", 0.0)
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["us"] for a in agg.values() if a["us"] == a["us"])
    print(f"{'kernel':58s} {'/step':>6s} {'us/launch':>11s} {'share':>6s} {'DRAM GB/launch (rd+wr)':>24s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        print(f"{k[:58]:58s} {a['n'] / steps:6.1f} {a['us'] / a['n']:11.1f} {100 * a['us'] / tot:5.1f}% "
              f"{a['rd'] / a['n'] / 1e9:11.4f} + {a['wr'] / a['n'] / 1e9:.4f}")
    print(f"total {tot / steps / 1e3:.3f} ms per factorization (serialized, cold-cache launches)")


if __name__ == "__main__":
    main()
