"""Per-unit throughput breakdown of the rectangle chain from an ncu raw page:
python tools/ncu_unit_breakdown.py gpurun_out/ncu_rect_raw.csv [n_kernels]
Prints, per kernel, every *_pct_of_peak_sustained_* metric >= 20 % (which
sub-unit the "L1/TEX Cache Throughput" / "Compute Throughput" headlines come
from) and the shared / global wavefront and sector counts."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hdr = rows[0]
data = [r for r in rows[1:] if r and r[0].isdigit()]
ki = hdr.index("Kernel Name")
counts = ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum",
          "smsp__inst_executed_op_shared_st.sum", "smsp__inst_executed_op_global_ld.sum",
          "smsp__inst_executed_op_global_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
          "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
          "lts__t_sectors.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
          "sm__cycles_elapsed.max", "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_sectors.sum",
          "l1tex__m_l1tex2xbar_write_sectors.sum", "smsp__inst_executed_op_local_ld.sum",
          "smsp__inst_executed_op_local_st.sum"]
for r in data[:nk]:
    print("==", r[ki].split("(")[0][:60])
    pct = []
    for h, v in zip(hdr, r):
        if "pct_of_peak" in h:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if x >= 20.0:
                pct.append((x, h))
    for x, h in sorted(pct, reverse=True):
        print(f"  {x:6.1f} %  {h}")
    for c in counts:
        if c in hdr:
            print(f"  {r[hdr.index(c)]:>16}  {c}")
