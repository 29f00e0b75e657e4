"""Summarise an ncu report: headline metrics + stall reasons (per issued instruction) per kernel."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = {
    "gpu__time_duration.sum": "duration",
    "sm__inst_executed.sum": "warp_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "launch__registers_per_thread": "regs",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "lsu_pipe_pct",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg": "lgds_wavefronts/SM",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_conflicts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_st_conflicts",
    "lts__t_bytes.sum": "l2_bytes",
}
for vals in rows[2:]:
    name = vals[hdr.index("Kernel Name")][:60]
    print("==", name)
    for k, nm in keys.items():
        if k in hdr:
            print(f"   {nm:18s} {vals[hdr.index(k)]} {rows[1][hdr.index(k)]}")
    st = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("   stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
