"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes) per kernel."""
import csv
import sys
from collections import defaultdict

UNIT = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    col = {h: i for i, h in enumerate(hdr)}
    k = defaultdict(dict)
    for r in rows[hi + 1:]:
        d = k[int(r[col["ID"]])]
        d["name"] = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        d["grid"] = r[col["Grid Size"]]
        d[r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", "")) * UNIT[r[col["Metric Unit"]]]
    return k


def main(path):
    k = load(path)
    tot, rd, wr, cnt = defaultdict(float), defaultdict(float), defaultdict(float), defaultdict(int)
    for d in k.values():
        n = d["name"]
        tot[n] += d["gpu__time_duration.sum"]
        rd[n] += d.get("dram__bytes_read.sum", 0)
        wr[n] += d.get("dram__bytes_write.sum", 0)
        cnt[n] += 1
    T = sum(tot.values())
    print(f"{'kernel':42s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>8s} {'dram_GB/s':>9s} {'rd_GB':>7s} {'wr_GB':>7s}")
    for n in sorted(tot, key=lambda n: -tot[n]):
        print(f"{n:42s} {cnt[n]:8d} {tot[n]/1e3:9.3f} {tot[n]/T:6.3f} {tot[n]/cnt[n]:8.2f} "
              f"{(rd[n]+wr[n])/tot[n]/1e3:9.1f} {rd[n]/1e9:7.3f} {wr[n]/1e9:7.3f}")
    print(f"{'total':42s} {sum(cnt.values()):8d} {T/1e3:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
