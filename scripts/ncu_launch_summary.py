"""Aggregates an ncu --csv metric log (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch) by kernel name:
launches, total time, DRAM bytes, achieved DRAM GB/s.

    python scripts/ncu_launch_summary.py gpurun_out/round_launches_c4_r08.csv
"""
import collections
import csv
import sys

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
         "GB": 1e9}
NS = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}


def summarize(path):
    hdr, per_launch = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].replace("<unnamed>::", "").replace("void ", "")
        name = name.split("(")[0].split("<")[0].split("::")[-1].strip()
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        per_launch.setdefault((d["ID"], name), {})[d["Metric Name"]] = v * (
            NS.get(u) or BYTES.get(u) or 1.0)
    agg = collections.OrderedDict()
    for (_, name), m in per_launch.items():
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    return agg


def main():
    for path in sys.argv[1:]:
        agg = summarize(path)
        total = sum(a[1] for a in agg.values())
        print(f"{path}: {sum(a[0] for a in agg.values())} launches, {total / 1e6:.3f} ms")
        print("| kernel | launches | total ms | share | DRAM GB | DRAM GB/s |")
        print("|---|---|---|---|---|---|")
        for name, (cnt, ns, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"| `{name}` | {cnt} | {ns / 1e6:.3f} | {ns / total:.1%} | {by / 1e9:.3f} | "
                  f"{by / ns if ns else 0:.0f} |")


if __name__ == "__main__":
    main()
