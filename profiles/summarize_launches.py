"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel share of a step."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            name = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("hpsg::", "")
            out.append((name, float(d["Metric Value"]) / 1000.0, d["Grid Size"]))
    return out


SETUP = ("k_insert", "k_fill_slots", "k_gen_keys", "k_scan<InsertScanOp>", "k_rows_non_finite")


def main(path, last=None):
    """Per-kernel share of the step: table setup (bulk inserts, key generation) excluded."""
    data = [d for d in load(path) if not d[0].startswith(SETUP)]
    if last:
        data = data[-last:]
    agg = collections.OrderedDict()
    for n, us, g in data:
        a = agg.setdefault(n, [0, 0.0, g])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'n':>4s} {'mean us':>9s} {'share':>7s}")
    for n, (c, us, g) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:60]:60s} {c:4d} {us / c:9.2f} {100 * us / tot:6.1f}%  grid={g}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
