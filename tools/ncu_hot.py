"""Per-address SASS hot spots of one kernel in an ncu report, grouped in address windows.
   python tools/ncu_hot.py rep.ncu-rep [window]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
win = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x100
base = int(rows[1][ia], 16)
tot = sum(int(r[iex]) for r in rows[1:])
stt = sum(int(r[ist]) for r in rows[1:])
agg = {}
for r in rows[1:]:
    off = int(r[ia], 16) - base
    key = off // win * win
    e = agg.setdefault(key, [0, 0, 0])
    e[0] += int(r[iex]); e[1] += int(r[ist]); e[2] += 1
print(f"total warp-instr {tot}, stall samples {stt}")
for k in sorted(agg):
    e = agg[k]
    if e[0] > tot * 0.01 or e[1] > stt * 0.01:
        print(f"{k:#07x}: instr {e[0]/tot*100:5.1f}%  stall {e[1]/stt*100:5.1f}%  ({e[2]} sass)")
