#!/bin/bash
# C4-path profile set: plain timing and one full ncu capture of consecutive staged row
# passes (sf_pass launches alternate pass A, pass B) in mid-sweep.
set -x
TAG=${1:-r02a}
NT=${2:-512}
SKIP=${3:-200}
mkdir -p gpurun_out
python tools/c4_probe.py 128 $NT 3 > gpurun_out/${TAG}_c4_probe.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:sf_pass --launch-skip $SKIP --launch-count 2 \
  -f -o gpurun_out/${TAG}_ncu_sf_pass python tools/c4_probe.py 128 $NT 1 > gpurun_out/${TAG}_ncu_sf_pass.log 2>&1
tail -3 gpurun_out/${TAG}_c4_probe.txt
