#!/bin/bash
# DRAM bytes of ONE K1 launch at the bench's full size (ncu, DRAM + time metrics only: one pass, no replay
# of the full section set).  usage (inside gpurun): tools/dram_bench.sh <config> <seeds> [--records]
# -> gpurun_out/k1_dram_bench_config<config>[_records].json
CFG=${1:-2}; SEEDS=${2:-2048}; EXTRA=$3
SUF=""; [ "$EXTRA" == "--records" ] && SUF="_records"
SER=""; [ "$CFG" == "2" ] && SER="--series"
OUT=gpurun_out/k1_dram_bench_config${CFG}${SUF}
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k1_simulate -c 1 --csv --log-file $OUT.csv python tools/profile_k1.py --config $CFG --seeds $SEEDS \
  $SER $EXTRA > $OUT.log 2>&1
python - "$OUT" "$CFG" <<'PY'
import csv, json, re, sys
out, cfg = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(out + ".csv")) if len(r) > 10]
h = rows[0]; im, iu, iv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
m = {r[im]: float(r[iv].replace(",", "")) * scale[r[iu]] for r in rows[1:]}
log = open(out + ".log").read()
g = re.search(r"replicas (\d+) des_events (\d+) msg_events (\d+).*flags (\d+) n_requests (\d+)", log)
d = {"config": cfg, "replicas": int(g.group(1)), "des_events": int(g.group(2)), "flags": int(g.group(4)),
     "n_requests": int(g.group(5)), "dram_bytes_read": m["dram__bytes_read.sum"],
     "dram_bytes_write": m["dram__bytes_write.sum"],
     "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
     "k1_seconds_under_ncu": m["gpu__time_duration.sum"],
     "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k1_simulate -c 1 "
            "python tools/profile_k1.py --config %d (bench size)" % cfg}
json.dump(d, open(out + ".json", "w"), indent=1)
print(json.dumps(d))
PY
