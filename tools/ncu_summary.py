"""Summarise an `ncu --csv` (long format) log: one line per launch."""
import csv
import sys
from collections import OrderedDict


def parse(path, pattern=""):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if pattern and pattern not in r["Kernel Name"]:
            continue
        key = (r["ID"], r["Kernel Name"])
        rows.setdefault(key, {"grid": r.get("Grid Size"), "block": r.get("Block Size")})
        try:
            rows[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            rows[key][r["Metric Name"]] = r["Metric Value"]
    return rows


if __name__ == "__main__":
    rows = parse(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
    for (i, name), m in rows.items():
        short = name.split("(")[0][-60:]
        dur = m.get("gpu__time_duration.sum", 0)
        rd = m.get("dram__bytes_read.sum", 0)
        wr = m.get("dram__bytes_write.sum", 0)
        pct = m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", "")
        print(f"{i:>4} {short:60s} grid={m['grid']:>14s} {dur/1e3:9.2f} us  rd={rd/1e6:9.2f} MB "
              f"wr={wr/1e6:8.2f} MB  {rd/dur if dur else 0:8.1f} GB/s  dram%={pct}")
