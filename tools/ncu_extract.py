"""Dev tool: per-kernel summary of an ncu report (.ncu-rep) -> markdown-ish lines.
usage: ncu -i REPORT --page raw --csv | python tools/ncu_extract.py"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[0]
units = rows[1]


def col(name):
    return h.index(name) if name in h else None


want = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes_srcunit_tex.sum", "l2<->sm bytes"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2->sm read sectors"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor hmma % elapsed"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_elapsed", "tensor hmma inst %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor mem cycles % elapsed"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "bf16 tensor ops % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]
name_i = col("Kernel Name")
for r in rows[2:]:
    if len(r) <= name_i:
        continue
    print(r[name_i][:90])
    for m, label in want:
        i = col(m)
        if i is not None and r[i] != "":
            print(f"    {label:32s} {r[i]} {units[i]}")
if "--list" in sys.argv:
    for i, c in enumerate(h):
        if any(k in c for k in ("tensor", "dram__bytes", "lts__t_bytes")):
            print(c, units[i])
