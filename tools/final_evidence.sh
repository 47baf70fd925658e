#!/bin/bash
# Evidence set tied to ONE build (run on the GPU box: bash tools/final_evidence.sh <tag>).
# The DRAM-traffic capture comes first so that profiles/ncu_sweep_c4.json carries this build's
# hash when the bench lines are taken; everything lands in gpurun_out/<tag>_* and is copied
# into profiles/ in the build container.
set -x
T=${1:-final}
O=gpurun_out
mkdir -p $O
H=$(python -c "import bench; print(bench.build_hash())")
echo $H > $O/${T}_build_hash.txt
python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/${T}_traffic_c4_apply.csv python tools/c4_probe.py 128 2048 1 > $O/${T}_ncu_traffic.log 2>&1
python tools/traffic_summary.py $O/${T}_traffic_c4_apply.csv $H $O/${T}_ncu_sweep_c4.json 790017291059.2 > /dev/null
sed -i "s#$O/${T}_traffic_c4_apply.csv#profiles/traffic_${T}_c4_apply.csv.gz#" $O/${T}_ncu_sweep_c4.json
cp $O/${T}_ncu_sweep_c4.json profiles/ncu_sweep_c4.json
python bench.py > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err
python bench.py --steps 10 --warmup 3 --config C2 > $O/${T}_bench_c2.json 2> $O/${T}_bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/${T}_bench_ref_c4.json 2> $O/${T}_bench_ref_c4.err
python tools/c3_probe.py 512 1024 > $O/${T}_c3_probe.txt 2>&1
python tools/c5_probe.py 256 16 > $O/${T}_c5_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 7000 --csv --log-file $O/${T}_launches_bench_c4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_bench.log 2>&1
tail -3 $O/${T}_gputest.log
