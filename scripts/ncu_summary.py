"""Text summary of the key ncu --set full metrics of one kernel capture (profiles/ evidence)."""
import csv, io, subprocess, sys

rep, name = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
keys = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed_pipe_xu.sum", "XU (MUFU) instructions"),
]
for v in rows[2:]:   # every matching launch of the report (e.g. the three GEMM epilogue variants)
    d = dict(zip(h, v))
    if name not in d.get("Kernel Name", ""):
        continue
    print(f"kernel: {d['Kernel Name'][:120]}")
    for k, label in keys:
        if k in d:
            print(f"  {label:32s} {d[k]:>18s} {dict(zip(h, u)).get(k, '')}")
    tensor = [k for k in h if "tensor" in k and "pct" in k]
    for k in tensor[:6]:
        print(f"  {k[:60]:60s} {d[k]}")
