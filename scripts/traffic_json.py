"""profiles/traffic.json from an ncu --set full report: per kernel (template
name as bench.py names it) dram bytes read + written per launch.
python scripts/traffic_json.py report.ncu-rep > profiles/traffic.json"""
import csv, json, re, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("tg::", "").replace(" ", "")
    name = re.sub(r"^k_fused_bottom<(\d+),(\d+).*>$", r"k_fused_bottom<\1,\2>", name)
    name = re.sub(r"<(\d+),.*>$", r"<\1>", name) if name.startswith("k_interp_top_smem") else name
    name = name.replace("<true>", "<1>").replace("<false>", "<0>")
    b = float(r[ri].replace(",", "")) * scale[units[ri]] + float(r[wi].replace(",", "")) * scale[units[wi]]
    res.setdefault(name, b)
json.dump(res, sys.stdout, indent=1)
