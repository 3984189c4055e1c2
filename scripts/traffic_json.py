"""Record one ncu report's K3 DRAM bytes into profiles/traffic.json (read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

w, batch, rep = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}


def metric(name):
    i = hdr.index(name)
    return float(vals[i].replace(",", "")) * scale.get(units[i], 1)


rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[w] = {"batch": batch, "kernel": vals[hdr.index("Kernel Name")][:80], "dram_read_bytes": rd,
           "dram_write_bytes": wr, "k3_dram_bytes_per_launch": rd + wr,
           "gpu_time_ns": metric("gpu__time_duration.sum"), "source": os.path.basename(rep)}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[w]))
