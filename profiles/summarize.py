"""Summarise ncu captures into profiles/<round>/ (run here, on the CPU box).

  python profiles/summarize.py <round> <config> <launches.csv> [<full.ncu-rep>]

launches.csv : `ncu --metrics gpu__time_duration.sum --clock-control none --csv`
               over `bench.py --steps K --warmup W --no-cpu-baseline`
full.ncu-rep : `ncu --set full --import-source on -k regex:... -c N` of the same command
Writes <round>/launches_<config>.md (per-kernel share of the step) and, with a
full capture, <round>/full_<config>.md plus the DRAM bytes per launch that
bench.py reports as roofline.traffic (profiles/ncu_traffic.json).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

# bench.py stage -> kernels whose DRAM traffic it sums
STAGE_KERNELS = {
    "bloom_scan": ["bloom_members", "members_compact"],
    "dec_bloom_scan": ["bloom_members", "members_compact"],
    "p2_sets": ["p2_pairs", "p2_scatter"],
    "dec_p2_sets": ["p2_pairs", "p2_scatter"],
    "topr": ["topr_hist", "topr_select"],
    "index": ["nz_count", "nz_write"],
    "p2_engine": ["p2_engine"],
    "dec_p2_engine": ["p2_engine"],
    "pack_crc": ["crc_chunks"],
    "dec_parse_crc": ["crc_chunks"],
}


def short(name):
    base = name.split("(")[0].replace("void ", "").strip()
    if "at::" in name or "elementwise_kernel" in name:
        return "[torch setup/flush, outside the timed events] " + base.split("::")[-1][:40]
    return base.split("::")[-1]


def launches(path, steps_hint=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(d["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"])
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return []
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9}
    res = []
    for r in rows[2:]:
        rec = {}
        for h, u, v in zip(hdr, units, r):
            x = num(v)
            rec[h] = (x * scale[u] if u in scale else x) if x is not None else v
        res.append(rec)
    return res


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    rnd, cfg, lpath = sys.argv[1], sys.argv[2], sys.argv[3]
    fpath = sys.argv[4] if len(sys.argv) > 4 else None
    outdir = os.path.join(HERE, rnd)
    os.makedirs(outdir, exist_ok=True)
    agg = launches(lpath)
    total = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list — bench.py --config {cfg} (cold-cache, serialised: compare SHARES)", "",
             f"source: `{os.path.basename(lpath)}`; total kernel time {total / 1e3:.1f} us over all captured steps", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / total:.1f}% |")
    open(os.path.join(outdir, f"launches_{cfg}.md"), "w").write("\n".join(lines) + "\n")
    if not fpath:
        return
    recs = full(fpath)
    keys = [("gpu__time_duration.sum", "duration ns"), ("dram__bytes_read.sum", "DRAM read B"),
            ("dram__bytes_write.sum", "DRAM write B"),
            ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem % peak"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
            ("launch__registers_per_thread", "regs"),
            ("smsp__inst_executed.sum", "warp instr")]
    lines = [f"# ncu --set full — bench.py --config {cfg}", "",
             "| kernel | " + " | ".join(v for _, v in keys) + " |", "|---" * (len(keys) + 1) + "|"]
    traffic = collections.defaultdict(list)
    instr = collections.defaultdict(list)
    for rec in recs:
        k = short(rec.get("Kernel Name", "?")).split("<")[0]
        vals = [f"{rec[m]:.4g}" if isinstance(rec.get(m), float) else str(rec.get(m, "")) for m, _ in keys]
        lines.append(f"| `{k}` | " + " | ".join(vals) + " |")
        rd, wr = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
        if isinstance(rd, float) and isinstance(wr, float):
            traffic[k].append(rd + wr)
        if isinstance(rec.get("smsp__inst_executed.sum"), float):
            instr[k].append(rec["smsp__inst_executed.sum"])
    open(os.path.join(outdir, f"full_{cfg}.md"), "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(HERE, "ncu_traffic.json")
    tab = json.load(open(tpath)) if os.path.exists(tpath) else {}
    per_stage = {}
    for stage, kernels in STAGE_KERNELS.items():
        parts = [sum(traffic[k]) / len(traffic[k]) for k in kernels if traffic.get(k)]
        if parts:
            per_stage[stage] = sum(parts)
    tab[cfg] = per_stage
    # warp instructions per launch of the stage's main kernel (the issue roofline)
    tab[cfg + ":warp_instr"] = {stage: sum(instr[k]) / len(instr[k]) for stage, kernels in STAGE_KERNELS.items()
                                for k in kernels[:1] if instr.get(k)}
    json.dump(tab, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
