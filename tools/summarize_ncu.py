"""Summarise an ncu --set full report (one or more kernels) into a JSON file for profiles/:
per kernel launch the duration, DRAM bytes, L2 bytes, tensor-pipe and DRAM utilisation."""
import csv, json, subprocess, sys
rep, out_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_active.avg",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors.sum"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = []
for vals in rows[2:]:
    d = {"kernel": vals[hdr.index("Kernel Name")][:90]}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            d[w] = f"{vals[i]} {units[i]}".strip()
    rb = float(vals[hdr.index("dram__bytes_read.sum")].replace(",", "")) * scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
    wb = float(vals[hdr.index("dram__bytes_write.sum")].replace(",", "")) * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
    d["dram_bytes_per_launch"] = rb + wb
    out.append(d)
json.dump(out, open(out_json, "w"), indent=1)
for d in out:
    print(d["kernel"][:60], d["gpu__time_duration.sum"], "dram", round(d["dram_bytes_per_launch"] / 1e6, 2), "MB",
          "tensor", d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
