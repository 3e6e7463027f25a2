"""Text summary of one ncu --set full capture for profiles/: key metrics, warp-stall shares,
top source lines.  python tools/ncu_report.py report.ncu-rep "header line" > profiles/xxx.txt"""
import csv, io, subprocess, sys
rep = sys.argv[1]
print("# " + (sys.argv[2] if len(sys.argv) > 2 else rep))
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    print("kernel:", d.get("Kernel Name"))
    for k in keys:
        if k in d:
            print(f"{k}: {d[k]} {u.get(k, '')}")
    stalls = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
    vals = [(float(d[k].replace(",", "")), k) for k in stalls if d.get(k)]
    tot = sum(v for v, _ in vals) or 1.0
    print("warp-stall samples (share):")
    for v, k in sorted(vals, reverse=True)[:10]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%")
print("top source lines (tools/ncu_lines.py):")
sys.stdout.flush()
subprocess.run([sys.executable, __file__.replace("ncu_report.py", "ncu_lines.py"), rep, "20"])
