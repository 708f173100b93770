#!/bin/bash
# On the GPU box: warp-state / scheduler / source-level stall sampling of the
# dominant latency-bound kernels of one FULL-size sort (application replay:
# the 31 GB C5 state is re-created per pass instead of saved per kernel).
# usage: bash tools/prof_stalls.sh PREFIX CONFIG
P=${1:-r02x}; CFG=${2:-c5_nodup}
mkdir -p gpurun_out
SECS="--section SpeedOfLight --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --section SourceCounters --section InstructionStats --section MemoryWorkloadAnalysis"
for spec in "k_step_cta<:1" "k_cta_sort<.int.4>:1" "k_cta_sort<.int.8>:1"; do
    k=${spec%%:*}; skip=${spec##*:}; tag=$(echo $k | tr -cd "a-z_0-9")
    timeout 1200 ncu --replay-mode application $SECS --clock-control none --import-source on \
        --kernel-name-base demangled -k "regex:s5g::${k}" --launch-skip $skip -c 1 -o /tmp/${P}_${tag} -f \
        python tools/one_sort.py --config $CFG > gpurun_out/${P}_${tag}_ncu.log 2>&1
    ncu -i /tmp/${P}_${tag}.ncu-rep --page details > gpurun_out/${P}_${tag}_details.txt 2>&1
    ncu -i /tmp/${P}_${tag}.ncu-rep --page source --csv --print-source sass > /tmp/${P}_${tag}_sass.csv 2>/dev/null
    python tools/sass_hot.py /tmp/${P}_${tag}_sass.csv > gpurun_out/${P}_${tag}_hot.txt 2>&1
    ncu -i /tmp/${P}_${tag}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${P}_${tag}_src.csv 2>/dev/null
done
