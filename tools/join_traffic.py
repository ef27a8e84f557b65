"""DRAM traffic of k_join from an ncu --metrics csv log: writes
profiles/join_traffic.json for bench.py's roofline.traffic.
usage: join_traffic.py <ncu.csv> <capture description>

Only k_join launches count (the kernel name "k_join<...>": not k_join_lists /
k_join_bits).  Under ncu's replay (memory save/restore) the offer-queue
budget can shrink and an iteration then runs as two slices, so the file
records DRAM bytes per millisecond of join time; bench.py multiplies it by
its own measured time per (unsliced) launch."""
import csv, json, os, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ik, im, iu, iv, iid = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                       h.index("Metric Value"), h.index("ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6,
         "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}
per = {}
for r in rows[1:]:
    if "k_join<" not in r[ik]:
        continue
    d = per.setdefault(r[iid], {})
    d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
L = list(per.values())
div = len(L)
rd = sum(d["dram__bytes_read.sum"] for d in L) / div
wr = sum(d["dram__bytes_write.sum"] for d in L) / div
ms = sum(d["gpu__time_duration.sum"] for d in L) / div
out = {"kernel": "k_join", "launches": len(L), "per": div, "capture": sys.argv[2],
       "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic_bytes": rd + wr,
       "duration_ms": ms, "per_launch": [{"read": d["dram__bytes_read.sum"],
                                          "write": d["dram__bytes_write.sum"],
                                          "ms": d["gpu__time_duration.sum"]} for d in L],
       "dram_bytes_per_ms": (rd + wr) / ms}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "join_traffic.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_launch"}))
