#!/bin/bash
# Round-end evidence set on one B200: tests, bench lines, ncu launch list and full captures,
# DRAM traffic of one apply, DMMA pipe counters, DGEMM peak, compute-sanitizer logs.
set -x
TAG=${1:-r02h}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_gputest.log
python bench.py --steps 5 --warmup 3 > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err
python bench.py --steps 10 --warmup 3 --config C2 > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref_c4.json 2> $O/${TAG}_bench_ref_c4.err
python tools/dgemm_peak.py > $O/${TAG}_dgemm_peak.txt 2>&1
for c in C2 C4 C3; do python tools/config_arnoldi.py $c > $O/${TAG}_arnoldi_$c.json 2> $O/${TAG}_arnoldi_$c.err; done
LRK_SF_TIMING=1 python tools/c4_probe.py 128 2048 1 > $O/${TAG}_sf_timing.txt 2>&1
python tools/c3_probe.py 512 1024 > $O/${TAG}_c3_probe.txt 2>&1
python tools/c5_probe.py 256 16 > $O/${TAG}_c5_probe.txt 2>&1
python tools/hbm_roofline.py > $O/${TAG}_streaming_kernels.jsonl 2>&1
# launch list of the bench command (first 7000 launches: setup + the first apply)
ncu --metrics gpu__time_duration.sum --clock-control none -c 7000 --csv --log-file $O/${TAG}_launches_bench_c4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_bench.log 2>&1
# DRAM traffic + time of every launch of one full C4 apply
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/${TAG}_traffic_c4_apply.csv python tools/c4_probe.py 128 2048 1 > $O/${TAG}_ncu_traffic.log 2>&1
python -c "import bench; print(bench.build_hash())" > $O/${TAG}_build_hash.txt
# full captures of pass A / pass B late in the forward sweep at full size (rank 18)
ncu --set full --clock-control none --import-source on -k regex:sf_pass --launch-skip 900 --launch-count 2 \
  -f -o $O/${TAG}_ncu_sf_pass python tools/c4_probe.py 128 2048 1 > $O/${TAG}_ncu_sf_pass.log 2>&1
# which counters see the FP64 tensor pipe
ncu --query-metrics 2>/dev/null | grep -i -E "dmma|pipe_fp64|pipe_tensor" > $O/${TAG}_metric_names.txt
# compute-sanitizer is closed on this pool (it answers with a refusal); keep the answer as the record
timeout 120 compute-sanitizer --tool memcheck python tools/sanitize_small.py > $O/${TAG}_sanitizer_memcheck.log 2>&1
echo "rc=$?" >> $O/${TAG}_sanitizer_memcheck.log
python tools/sanitize_small.py > $O/${TAG}_sanitize_small_plain.log 2>&1
tail -3 $O/${TAG}_gputest.log
