"""Summarise an ncu --set full capture (one kernel launch) into a JSON for profiles/:
duration, DRAM bytes read+written (the `traffic` of bench.py's roofline), throughputs and the
tensor-pipe activity.   python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/x.json"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "Kernel Name": "kernel",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
res = {}
for i, name in enumerate(hdr):
    if name in want:
        v = vals[i].replace(",", "")
        try:
            f = float(v) * scale.get(units[i], 1.0)
            res[want[name]] = f
            res[want[name] + "_raw"] = f"{vals[i]} {units[i]}"
        except ValueError:
            res[want[name]] = vals[i]
if "dram_read" in res and "dram_write" in res:
    res["dram_bytes_per_launch"] = res["dram_read"] + res["dram_write"]
res["source"] = f"ncu --set full --clock-control none, {rep}"
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
