"""One line per profiled kernel of an ncu report: duration, DRAM / memory / SM throughput,
occupancy, grid.  Usage: python tools/ncu_table.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Grid Size", "Block Size", "Registers Per Thread"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    rows = {}
    for row in r:
        if row[mi] in WANT:
            d = rows.setdefault(row[ii], {"name": row[ki]})
            key = row[mi] + (" GB/s" if row[ui] == "Gbyte/s" else "")
            d.setdefault(key, row[vi])
    print(f"{'id':>3} {'us':>8} {'dram%':>6} {'mem%':>6} {'sm%':>6} {'occ%':>6} {'grid':>6} {'blk':>5}  kernel")
    for i, d in sorted(rows.items(), key=lambda kv: int(kv[0])):
        print(f"{i:>3} {d.get('Duration', ''):>8} {d.get('DRAM Throughput', ''):>6} {d.get('Memory Throughput', ''):>6} "
              f"{d.get('Compute (SM) Throughput', ''):>6} {d.get('Achieved Occupancy', ''):>6} {d.get('Grid Size', ''):>6} "
              f"{d.get('Block Size', ''):>5}  {d['name'][:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
