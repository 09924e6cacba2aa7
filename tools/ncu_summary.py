"""Summarise an ncu report: key throughput metrics per kernel and the top
stalled SASS lines (mbarrier waits resolved to names when a barrier map is given)."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = [r"^Kernel Name$", r"^gpu__time_duration.sum$", r"^dram__bytes_(read|write).sum$",
        r"^sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active$",
        r"^sm__inst_executed_pipe_(xu|fma|alu|lsu).avg.pct_of_peak_sustained_active$",
        r"^sm__issue_active.avg.pct_of_peak_sustained_elapsed$",
        r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^dram__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^launch__(registers_per_thread|grid_size|block_size)$",
        r"^sm__cycles_elapsed.avg.per_second$",
        r"^l1tex__throughput.avg.pct_of_peak_sustained_active$",
        r"^l1tex__data_pipe_(tc|lsu)_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed$",
        r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$",
        r"^l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_red.sum$",
        r"^l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum$"]
for r in rows[2:]:
    print("----")
    for i, h in enumerate(hdr):
        if any(re.search(w, h) for w in want):
            print(f"  {h} = {r[i]} {units[i]}")
