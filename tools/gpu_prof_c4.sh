#!/bin/bash
# C4-path profile set: plain timing, ncu launch list, full captures of the two staged row passes.
set -x
TAG=${1:-r02a}
mkdir -p gpurun_out
python tools/c4_probe.py 128 512 3 > gpurun_out/${TAG}_c4_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python tools/c4_probe.py 128 128 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
for k in sf_update_project sf_subtract; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 41 --launch-count 2 \
    -f -o gpurun_out/${TAG}_ncu_$k python tools/c4_probe.py 128 128 1 > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
tail -3 gpurun_out/${TAG}_c4_probe.txt
