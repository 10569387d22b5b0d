"""Write a compact, committed summary of an ncu --set full report.
    python tools/ncu_summary.py <report.ncu-rep> <cells> <algorithmic_bytes_per_cell> <out.txt>"""
import csv, io, json, subprocess, sys
rep, cells, bpc, out = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
m = dict(zip(rows[0], rows[2]))
u = dict(zip(rows[0], rows[1]))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__cycles_active.avg", "sm__cycles_active.max", "smsp__inst_executed.sum",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_bytes.sum"]
lines = [f"ncu --set full summary of {rep.split('/')[-1]}"]
for k in keys:
    if k in m:
        lines.append(f"  {k:62s} {m[k]} {u.get(k, '')}")
def num(k, scale=1.0):
    try:
        return float(m[k].replace(",", "")) * scale
    except Exception:
        return None
t_ms = num("gpu__time_duration.sum")
unit_t = u.get("gpu__time_duration.sum", "")
t_s = t_ms * (1e-3 if unit_t == "ms" else 1e-6 if unit_t == "us" else 1e-9 if unit_t == "ns" else 1.0)
def gb(k):
    v = num(k)
    un = u.get(k, "")
    return v * {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "Tbyte": 1e3}.get(un, 1.0)
rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
alg = cells * bpc / 1e9
lines.append(f"  cells per launch {cells:.0f}; algorithmic bytes {alg:.3f} GB ({bpc:.0f} B/cell); "
             f"DRAM traffic {rd + wr:.3f} GB ({(rd + wr) / alg:.2f}x algorithmic)")
lines.append(f"  duration {t_s * 1e3:.3f} ms -> algorithmic {alg / t_s:.0f} GB/s; DRAM {(rd + wr) / t_s:.0f} GB/s")
warp_inst = num("smsp__inst_executed.sum")
if warp_inst:
    lines.append(f"  thread instructions per cell: {warp_inst * 32 / cells:.1f}")
stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: num(k) for k in m
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
stalls = {k: v for k, v in stalls.items() if v}
if stalls:
    tot = sum(stalls.values())
    lines.append("warp-state samples (smsp__pcsamp_warps_issue_stalled_*, share of all samples):")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        lines.append(f"  {k:28s}{100 * v / tot:5.1f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
print(json.dumps({"traffic_GB_per_launch": rd + wr}))
