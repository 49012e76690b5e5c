"""Summarise an ncu report: headline metrics, stall reasons, hot SASS segments."""
import csv, subprocess, sys, io

rep = sys.argv[1]
kid = int(sys.argv[3]) if len(sys.argv) > 3 else 0
def page(*a):
    out = subprocess.run(["ncu", "-i", rep, *a, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

raw = page("--page", "raw")
h, v = raw[0], raw[2 + kid]
print("kernel:", v[h.index("Kernel Name")][:100])
d = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for k in keys:
    print(f"{k:60s} {d.get(k)}")
st = {k: float(d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
print("stalls per issue:", ", ".join(f"{k[34:-27]} {x:.2f}" for k, x in sorted(st.items(), key=lambda t: -t[1])[:9]))
if len(sys.argv) > 2:
    rows = page("--page", "source", "--print-source", "sass")
    hdr, data = rows[1], rows[2:]
    ia, isrc, iad, ist = (hdr.index(x) for x in ("Instructions Executed", "Source", "Address", "Warp Stall Sampling (All Samples)"))
    tot = sum(int(r[ia] or 0) for r in data)
    segs, cur = [], None
    for r in data:
        n = int(r[ia] or 0)
        if cur and cur[0] == n:
            cur[2].append(r)
        else:
            cur = [n, r[iad], [r]]
            segs.append(cur)
    segs.sort(key=lambda s: -s[0] * len(s[2]))
    for n, a, rs in segs[: int(sys.argv[2])]:
        print(a[-5:], n, len(rs), f"{n*len(rs)/tot*100:.1f}%", "stall", sum(int(x[ist] or 0) for x in rs), rs[0][isrc][:50])
    print("top stalled instructions:")
    for r in sorted(data, key=lambda r: -int(r[ist] or 0))[:12]:
        print(" ", r[iad][-5:], r[ist], r[isrc][:80])
