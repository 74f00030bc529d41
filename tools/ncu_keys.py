"""Key metrics of `ncu --page raw --csv` exports (one kernel each) as a JSON table:
python tools/ncu_keys.py profiles/r02/full_*.raw.csv > profiles/r02/ncu_full_summary.json"""
import csv
import json
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_active_pct",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed": "utchmma_ops_pct_of_peak",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_to_tc_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
}
out = {}
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")][:90] if "Kernel Name" in h else ""}
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            d[name] = f"{v[i]} {u[i]}".strip()
    out[path.split("/")[-1].replace(".raw.csv", "")] = d
print(json.dumps(out, indent=1))
