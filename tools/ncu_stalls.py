"""Top SASS stall sites of one kernel: python tools/ncu_stalls.py rep.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2], "-c", "1"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out))]
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(hdr) == len(r) and r[hdr.index("Address")].startswith("0x")]
ia, isrc, ist, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                               "Instructions Executed"))
num = lambda s: float(s.replace(",", "") or 0)
tot = sum(num(r[ist]) for r in data) or 1
tex = sum(num(r[iex]) for r in data) or 1
print(f"warp instr {tex:.3e}; stall samples {tot:.0f}")
for r in sorted(data, key=lambda r: -num(r[ist]))[: int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{r[ia]}  stall {num(r[ist]) / tot * 100:5.1f}%  {r[isrc][:90]}")
if len(sys.argv) > 4:  # window around an address: ... <addr-hex> 
    a0 = int(sys.argv[4], 16)
    seen = set()
    for r in data:
        a = int(r[ia], 16)
        if abs(a - a0) <= 0x200 and a not in seen:
            seen.add(a)
            print(f"{r[ia]}  {num(r[ist]) / tot * 100:5.1f}%  {r[isrc][:100]}")
