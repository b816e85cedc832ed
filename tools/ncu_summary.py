"""Summarise an ncu --set full report: key throughput metrics + top stall sites.
  python tools/ncu_summary.py gpurun_out/x.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
        "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_issue_stalled", "sm__inst_executed_pipe_uniform",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for i, name in enumerate(h):
    if name in want or any(name.startswith(w) and "pct" in name and "smsp__pcsamp" in name for w in want):
        print(f"{name}: {v[i]} {u[i]}")
# stall reasons
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and name.endswith("_not_issued") is False and "ratio" not in name:
        try:
            if float(v[i]) > 0:
                pass
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[si] or 0) for x in data if x[si] not in ("", "-"))
print(f"--- top {ntop} SASS sites by stall samples (total {tot:.0f})")
for x in sorted(data, key=lambda x: -float(x[si] or 0))[:ntop]:
    print(f"{float(x[si]) / tot * 100:5.1f}% {x[0][-5:]} {x[1][:100]}")
