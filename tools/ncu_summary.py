"""Key metrics of an ncu --set full report (raw page) + top stall reasons + top source lines."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, units, vals = r[0], r[1], r[2]
d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
print("kernel:", d.get("Kernel Name", ("", ""))[1])
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x"]
for k in keys:
    if k in d:
        print(f"  {k:90s} {d[k][1]:>14s} {d[k][0]}")
st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
      for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stall reasons (share of samples):")
for h, v in sorted(st, key=lambda x: -x[1])[:8]:
    print(f"  {h:40s} {100 * v / tot:5.1f}%")
