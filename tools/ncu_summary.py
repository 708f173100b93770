"""Summarise an `ncu --set full` capture of one sort (bench.py --steps 1
--warmup 0): per-kernel launches, time, DRAM bytes and occupancy/issue, as
the committed profiles/<round>_ncu_kernels.csv and the traffic JSON that
bench.py's roofline.traffic reads.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
col = {k: i for i, k in enumerate(h)}
keep = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        # warp divergence (threads active per issued instruction, of 32) and
        # global-access sector efficiency (sectors per request, 4 = a fully
        # used 128-byte line per warp request of 4-byte words)
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]
keep_missing = []
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0,
         "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "ns": 1e-6}


def val(r, k):
    v = float(r[col[k]].replace(",", ""))
    return v * scale.get(units[col[k]], 1.0)


keep_missing = [k for k in keep if k not in col]
keep = [k for k in keep if k in col]
with open(prefix + "_ncu_kernels.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(keep)
    w.writerow([units[col[k]] for k in keep])
    for r in data:
        w.writerow([r[col[k]] for k in keep])
kern = {}
for r in data:
    name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("s5g::", "")
    name = re.sub(r"\(int\)|\(bool\)", "", name)
    e = kern.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "ms": 0.0, "warp_inst": 0.0,
                               "thread_inst": 0.0, "ld_sec": 0.0, "ld_req": 0.0, "st_sec": 0.0,
                               "st_req": 0.0})
    e["launches"] += 1
    wi = val(r, "smsp__inst_executed.sum")
    if "smsp__thread_inst_executed_per_inst_executed.ratio" in col:
        e["thread_inst"] += wi * val(r, "smsp__thread_inst_executed_per_inst_executed.ratio")
    for k2, m in (("ld_sec", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
                  ("ld_req", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
                  ("st_sec", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum"),
                  ("st_req", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum")):
        if m in col:
            e[k2] += val(r, m)
    e["dram_bytes"] += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    e["ms"] += val(r, "gpu__time_duration.sum")
    e["warp_inst"] += val(r, "smsp__inst_executed.sum")
for e in kern.values():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
    e["warp_inst_per_launch"] = e["warp_inst"] / e["launches"]
    e["threads_per_warp_inst"] = e["thread_inst"] / e["warp_inst"] if e["warp_inst"] else None
    e["ld_sectors_per_request"] = e["ld_sec"] / e["ld_req"] if e["ld_req"] else None
    e["st_sectors_per_request"] = e["st_sec"] / e["st_req"] if e["st_req"] else None
src = sys.argv[3] if len(sys.argv) > 3 else "one sort (tools/one_sort.py)"
json.dump({"source": f"ncu --set full, {src}, {prefix}_ncu_kernels.csv",
           "missing_metrics": keep_missing, "kernels": kern},
          open(prefix + "_traffic.json", "w"), indent=1)
print(f"{'kernel':28s} {'n':>3s} {'ms':>8s} {'DRAM GB':>8s} {'thr/inst':>8s} {'ld s/r':>7s} {'st s/r':>7s}")
for k, e in sorted(kern.items(), key=lambda x: -x[1]["ms"]):
    f = lambda x: f"{x:7.2f}" if x is not None else "    n/a"  # noqa: E731
    print(f"{k:28s} {e['launches']:3d} {e['ms']:8.3f} {e['dram_bytes'] / 1e9:8.3f} "
          f"{f(e['threads_per_warp_inst'])} {f(e['ld_sectors_per_request'])} "
          f"{f(e['st_sectors_per_request'])}")
