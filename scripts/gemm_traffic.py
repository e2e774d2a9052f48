"""K2 DRAM traffic vs algorithmic bytes (bench roofline.traffic): parse the ncu
launch list of `scripts/profile_step.py` and write profiles/r02_gemm_traffic.json.

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --cache-control none -k regex:sk_gemm --csv --log-file gpurun_out/gemm_traffic.csv \
        python scripts/profile_step.py --steps 2 > gpurun_out/traffic.log
    python scripts/gemm_traffic.py gpurun_out/gemm_traffic.csv gpurun_out/traffic.log
"""
import csv
import json
import os
import re
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
per = {}
for r in rows:
    per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * (
        {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(r["Metric Unit"], 1.0))
n = len(per)
rd = sum(v["dram__bytes_read.sum"] for v in per.values()) / n
wr = sum(v["dram__bytes_write.sum"] for v in per.values()) / n
alg = float(re.search(r"algorithmic_bytes_per_launch=(\d+)", open(sys.argv[2]).read()).group(1))
out = {"kernel": "sk_gemm_kernel",
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none "
                 "-k regex:sk_gemm, python scripts/profile_step.py --steps 2 --draft-model none (7B, 8 stages, bench workload; target GEMMs only)",
       "launches": n, "dram_read_bytes_per_launch": round(rd), "dram_write_bytes_per_launch": round(wr),
       "traffic_bytes_per_launch": round(rd + wr), "algorithmic_bytes_per_launch": round(alg),
       "traffic_over_algorithmic": round((rd + wr) / alg, 3),
       "note": "per-launch means over the same launches; write traffic = stream-K partials + epilogue outputs"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "r02_gemm_traffic.json"), "w"), indent=1)
print(json.dumps(out))
