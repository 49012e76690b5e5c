"""Instructions executed per CUDA source line of an ncu report (needs -lineinfo and
--import-source on), normalised by a unit count: python tools/ncu_lines.py rep.ncu-rep UNITS [N]

Sums the SASS rows that ncu lists under each CUDA line (the CUDA rows themselves are not
reliably CSV-escaped)."""
import csv, io, os, subprocess, sys

rep, units = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
acc, fname, hdr, cur = {}, "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0]:
        cur = f"{fname}:{r[0]}"
        acc.setdefault(cur, [0.0, 0, r[1][:80]])
    elif hdr and cur and len(r) == len(hdr) and r[2].startswith("0x"):
        a = acc[cur]
        a[0] += float(r[hdr.index("Instructions Executed")] or 0)
        a[1] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
tot = sum(a[0] for a in acc.values())
stt = sum(a[1] for a in acc.values()) or 1
print(f"total {tot:.4g} warp-instr, {tot / units:.4f} per unit")
for where, (v, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{where:>24} {v / units:8.4f} {100 * v / tot:5.1f}%  stall {100 * s / stt:5.1f}%  {src.strip()[:70]}")
