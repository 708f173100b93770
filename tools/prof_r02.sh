#!/bin/bash
# On the GPU box: per-kernel launch list of one full-size sort of a config
# (gpu__time_duration only: one pass, no replay of the 31 GB C5 state) and
# an ncu --set full capture of one sort at a scale ncu can replay, summarised
# there (divergence, sector efficiency, DRAM bytes per kernel).
# usage: bash tools/prof_r02.sh PREFIX CONFIG FULL_SCALE
P=${1:-r02x}; CFG=${2:-c5_nodup}; FS=${3:-0.0625}
mkdir -p gpurun_out
python tools/one_sort.py --config $CFG > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${P}_ncu_launches.csv python tools/one_sort.py --config $CFG > gpurun_out/${P}_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -o /tmp/${P}_full -f \
    python tools/one_sort.py --config $CFG --scale $FS > gpurun_out/${P}_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/${P}_full.ncu-rep gpurun_out/${P} "one $CFG sort at scale $FS (tools/one_sort.py)" \
    > gpurun_out/${P}_ncu_summary.txt 2>&1
for k in k_cta_sort k_scatter k_warp_sort k_classify k_step_cta; do
    ncu -i /tmp/${P}_full.ncu-rep --page source --csv --print-source sass -k regex:$k > /tmp/${P}_${k}_sass.csv 2>/dev/null
    python tools/sass_hot.py /tmp/${P}_${k}_sass.csv > gpurun_out/${P}_${k}_hot.txt 2>&1
done
