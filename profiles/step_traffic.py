"""Per-step DRAM traffic of the training step from an ncu capture (tracked evidence for
bench.py's roofline.traffic).

Input: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--clock-control none --csv -k regex:"k_"` over `bench.py --no-graph --pool 1 ...` (eager
steps; ncu serialises kernels and flushes caches between them, so these are COLD bytes per
launch, an upper bound on the in-graph traffic). The kernels of one training step are the
launches between two consecutive step starts that include a reduce; a step starts at the
training probe (k_probe), or, for insert-on-miss tables (config 5), at the insert's claim
(k_insert_claim: the insert pass writes the training record itself, no k_probe).
Usage: python profiles/step_traffic.py CSV WORKLOAD OUT_JSON
"""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("hpsg::", "")
        k = (d["ID"], name)
        rec = out.setdefault(k, {"name": name})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        if d["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            rec[d["Metric Name"]] = v * scale
        else:
            rec["us"] = v / 1000.0 if unit in ("nsecond", "ns") else v
    return list(out.values())


def steps(recs):
    """Split the launch list into training steps: each starts at a k_probe or k_insert_claim and
    must contain a reduce."""
    start = ("k_probe", "k_insert_claim")
    cur, out = [], []
    for r in recs:
        if r["name"].startswith(start) and cur:
            out.append(cur)
            cur = []
        cur.append(r)
    if cur:
        out.append(cur)
    return [s for s in out if s[0]["name"].startswith(start) and any("reduce" in r["name"] for r in s)]


def main(path, workload, out_path):
    st = steps(load(path))
    assert st, "no complete training step in the capture"
    s = st[-1]
    per = collections.OrderedDict()
    for r in s:
        a = per.setdefault(r["name"], {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "us": 0.0})
        a["launches"] += 1
        a["dram_read"] += r.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += r.get("dram__bytes_write.sum", 0.0)
        a["us"] += r.get("us", 0.0)
    tot_r = sum(a["dram_read"] for a in per.values())
    tot_w = sum(a["dram_write"] for a in per.values())
    doc = {}
    try:
        doc = json.load(open(out_path))
    except Exception:
        pass
    doc[workload] = {"source": path, "dram_read": int(tot_r), "dram_write": int(tot_w),
                     "serialized_us": round(sum(a["us"] for a in per.values()), 2),
                     "kernels": {k: {"launches": v["launches"], "dram_read": int(v["dram_read"]),
                                     "dram_write": int(v["dram_write"]), "us": round(v["us"], 2)}
                                 for k, v in per.items()}}
    json.dump(doc, open(out_path, "w"), indent=1)
    print(json.dumps({workload: {k: doc[workload][k] for k in ("dram_read", "dram_write", "serialized_us")}}))


if __name__ == "__main__":
    main(*sys.argv[1:4])
