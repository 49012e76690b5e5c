"""Turn an ncu --set full capture of the fused sweep into the committed evidence:
profiles/ncu_traffic.json (dram bytes per launch, read by bench.py's roofline.traffic)
and a short text summary.  Usage: python tools/ncu_to_profile.py REPORT KERNEL_LABEL OUT_TXT"""
import csv, io, json, os, subprocess, sys

rep, label, out_txt = sys.argv[1], sys.argv[2], sys.argv[3]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, v = raw[0], raw[2]
d = dict(zip(h, v))
num = lambda k: float(d[k].replace(",", ""))
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
ur, uw = raw[1][h.index("dram__bytes_read.sum")], raw[1][h.index("dram__bytes_write.sum")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale[ur]; wr *= scale[uw]
dur_ms = num("gpu__time_duration.sum") * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[raw[1][h.index("gpu__time_duration.sum")]]
path = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
cur = json.load(open(path)) if os.path.exists(path) else {}
cur[label] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "duration_ms_ncu": dur_ms,
              "source": os.path.basename(rep)}
json.dump(cur, open(path, "w"), indent=1)
st = {k: float(d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
lines = [f"kernel: {v[h.index('Kernel Name')]}", f"report: {os.path.basename(rep)} (ncu --set full --clock-control none)",
         f"duration_ms (ncu, serialized): {dur_ms:.4f}", f"dram_read_bytes: {rd:.0f}", f"dram_write_bytes: {wr:.0f}",
         f"instructions_executed: {num('smsp__inst_executed.sum'):.0f}",
         f"ipc_active: {num('sm__inst_executed.avg.per_cycle_active'):.2f}",
         f"issue_slots_busy_pct: {num('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}",
         f"registers_per_thread: {d.get('launch__registers_per_thread')}",
         f"warps_active_per_sm: {num('sm__warps_active.avg.per_cycle_active'):.1f}",
         "stalls_per_issue: " + ", ".join(f"{k[34:-27]} {x:.2f}" for k, x in sorted(st.items(), key=lambda t: -t[1])[:8])]
open(out_txt, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
