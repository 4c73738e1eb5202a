"""Summarise a K1 `ncu --set full` capture (tools/profile_k1.py) into profiles/<dir>/k1_ncu_summary.json.
usage: python tools/ncu_summary.py <report.ncu-rep> <profile_k1 log> <out.json> [config label]"""
import csv
import io
import json
import re
import subprocess
import sys

rep, log, out = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"]
keys += [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
d = {k: v[h.index(k)] for k in keys if k in h}
d["units"] = {k: u[h.index(k)] for k in keys if k in h}
m = re.search(r"replicas (\d+) des_events (\d+) msg_events (\d+)", open(log).read())
R, des = int(m.group(1)), int(m.group(2))
cfg = sys.argv[4] if len(sys.argv) > 4 else "config-2"
d["workload"] = "tools/profile_k1.py: " + cfg + " grid, %d replicas x 1000 requests, %d DES events (1 launch)" % (R, des)
d["warp_instr_per_des_event"] = float(d["smsp__inst_executed.sum"]) / des
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
dram = sum(float(d[k]) * scale[d["units"][k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
d["dram_bytes_per_des_event"] = dram / des
json.dump(d, open(out, "w"), indent=1)
print(json.dumps({k: d[k] for k in ("gpu__time_duration.sum", "warp_instr_per_des_event", "dram_bytes_per_des_event",
                                    "smsp__issue_active.avg.pct_of_peak_sustained_active")}))
