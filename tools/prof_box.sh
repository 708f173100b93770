#!/bin/bash
# On the GPU box: launch list of bench.py + ncu --set full of one C2 sort,
# summarised there (the .ncu-rep itself is too large to bring back).
# usage: bash tools/prof_box.sh PREFIX   (e.g. r01e)
P=${1:-rXX}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 > gpurun_out/${P}_bench_plain.jsonl 2> gpurun_out/${P}_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${P}_ncu_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${P}_ncu_l.log 2>&1
python tools/one_sort.py > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -o /tmp/${P}_full -f python tools/one_sort.py > gpurun_out/${P}_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/${P}_full.ncu-rep gpurun_out/${P} > gpurun_out/${P}_ncu_summary.txt 2>&1
for k in k_cta_sort k_scatter k_warp_sort k_classify k_step_cta; do
    ncu -i /tmp/${P}_full.ncu-rep --page source --csv --print-source sass -k regex:$k > /tmp/${P}_${k}_sass.csv 2>/dev/null
    python tools/sass_hot.py /tmp/${P}_${k}_sass.csv > gpurun_out/${P}_${k}_hot.txt 2>&1
done
