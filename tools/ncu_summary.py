"""Summarise an ncu report (--set full) into profiles/<round>/ncu_summary.json."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in WANT.items():
            if k in d:
                v = d[k].replace(",", "")
                try:
                    item[name] = float(v)
                except ValueError:
                    item[name] = v
                u = units[hdr.index(k)]
                if u in ("Kbyte", "Mbyte", "Gbyte", "byte") and isinstance(item[name], float):
                    item[name] *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if u == "usecond" or u == "us":
                    item[name] *= 1e3
                if u == "msecond" or u == "ms":
                    item[name] *= 1e6
        res.append(item)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
