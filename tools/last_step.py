"""Per-kernel durations of the last bench step in an ncu launch list: python tools/last_step.py l.csv [first-kernel]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
first = sys.argv[2] if len(sys.argv) > 2 else "topr_hist"
hdr, seq = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
        seq.append((k, float(d["Metric Value"]) / 1e3))
idx = [i for i, (k, _) in enumerate(seq) if k.startswith(first)]
last = seq[idx[-1]:] if idx else seq
print("total us", round(sum(v for _, v in last), 1), "kernels", len(last))
for k, v in last:
    print(f"{v:8.1f} {k}")
