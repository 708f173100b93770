#!/bin/bash
# On the GPU box: the round's evidence for one workload.
#  1. bench line (driver's settings) and the reference arm;
#  2. ncu launch list of one FULL-size sort with time + DRAM bytes per launch
#     (one pass, no replay) -> the traffic JSON bench.py reads;
#  3. ncu --set full of one sort at a scale ncu can replay -> divergence,
#     sector efficiency, issue / occupancy per kernel, SASS hot spots.
# usage: bash tools/prof_r02.sh PREFIX CONFIG FULL_SET_SCALE
P=${1:-r02x}; CFG=${2:-c5_nodup}; FS=${3:-0.0625}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/${P}_bench.jsonl 2> gpurun_out/${P}_bench.err || exit 1
python bench.py --config $CFG --impl reference --steps 3 --warmup 1 > gpurun_out/${P}_bench_reference.jsonl 2>&1
python tools/one_sort.py --config $CFG > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${P}_ncu_launches.csv python tools/one_sort.py --config $CFG > gpurun_out/${P}_ncu_l.log 2>&1
python tools/launch_traffic.py gpurun_out/${P}_ncu_launches.csv gpurun_out/${P}_${CFG}_traffic.json \
    "one full-size $CFG sort (tools/one_sort.py)" > gpurun_out/${P}_ncu_launches_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -o /tmp/${P}_full -f \
    python tools/one_sort.py --config $CFG --scale $FS > gpurun_out/${P}_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/${P}_full.ncu-rep gpurun_out/${P}_full "one $CFG sort at scale $FS (tools/one_sort.py)" \
    > gpurun_out/${P}_ncu_full_summary.txt 2>&1
ncu -i /tmp/${P}_full.ncu-rep --page source --csv --print-source sass > /tmp/${P}_sass.csv 2>/dev/null
for k in k_cta_sort k_scatter k_classify k_step_cta; do
    python tools/sass_hot.py /tmp/${P}_sass.csv $k > gpurun_out/${P}_${k}_hot.txt 2>&1
done
