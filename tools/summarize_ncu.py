"""Summarise an ncu --set full report of one kernel into a small text/JSON file for profiles/."""
import csv, json, subprocess, sys
rep, out_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_active.avg"]
d = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        d[w] = {"value": vals[i], "unit": units[i]}
rb = float(d["dram__bytes_read.sum"]["value"].replace(",", ""))
unit = d["dram__bytes_read.sum"]["unit"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
wb = float(d["dram__bytes_write.sum"]["value"].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["dram__bytes_write.sum"]["unit"]]
d["dram_bytes_per_launch"] = rb * scale + wb
json.dump(d, open(out_json, "w"), indent=1)
print(json.dumps(d, indent=1))
