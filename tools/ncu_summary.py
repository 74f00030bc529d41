"""Summarise an ncu report (--set full) into profiles/<round>/ncu_summary.json.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--map step_map.json]

With ``--map`` (written by tools/ncu_step.py) every profiled launch is attributed, in
launch order, to the step op that issued it, and per-kind totals are added under
``"by_kind"`` (bench.py reads them for ``roofline.traffic``)."""
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


def main(rep, out, map_path=None):
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
    if map_path is None:
        json.dump(res, open(out, "w"), indent=1)
        print(json.dumps(res, indent=1))
        return
    calls = json.load(open(map_path))
    i = 0
    for c in calls:
        for _ in range(c["kernels"]):
            if i < len(res):
                res[i].update(kind=c["kind"], layer=c["layer"])
            i += 1
    by = {}
    for c in calls:
        b = by.setdefault(c["kind"], {"calls": 0, "kernels": 0, "flops": 0.0, "alg_bytes": 0.0, "duration_ns": 0.0,
                                      "dram_read_bytes": 0.0, "dram_write_bytes": 0.0})
        b["calls"] += 1
        b["flops"] += c["flops"]
        b["alg_bytes"] += c["bytes"]
    for r in res:
        b = by.get(r.get("kind"))
        if b is None:
            continue
        b["kernels"] += 1
        for k in ("duration_ns", "dram_read_bytes", "dram_write_bytes"):
            if isinstance(r.get(k), float):
                b[k] += r[k]
    for b in by.values():
        b["dram_bytes_per_call"] = (b["dram_read_bytes"] + b["dram_write_bytes"]) / max(b["calls"], 1)
        b["alg_bytes_per_call"] = b["alg_bytes"] / max(b["calls"], 1)
    doc = {"launches": res, "by_kind": by, "matched": i == len(res), "n_profiled": len(res), "n_mapped": i}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(by, indent=1))
    print("matched", i, len(res))


if __name__ == "__main__":
    args = sys.argv[1:]
    mp = None
    if "--map" in args:
        j = args.index("--map")
        mp = args[j + 1]
        del args[j : j + 2]
    main(args[0], args[1], mp)
