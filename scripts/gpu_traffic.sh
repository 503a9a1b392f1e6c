#!/bin/bash
# Per-class DRAM traffic + tensor-pipe probes of every config (the tail of gpu_final.sh on its own).
TAG=${1:-traffic}
mkdir -p gpurun_out/$TAG
for C in C2 C3 C4 C5 S1; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none \
    --csv --log-file gpurun_out/traffic_$C.csv python scripts/traffic_probe.py --config $C > gpurun_out/$TAG/traffic_$C.log 2>&1
done
ls gpurun_out/traffic_*.csv
