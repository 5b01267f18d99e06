#!/bin/bash
# Round 2, final session: smoke, the full GPU suite, bench lines for every workload and the
# reference arm, ncu launch lists (config 3, config 2, config 4), sanitizers on the changed kernels.
set -x
TAG=r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke $? >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_$TAG.log 2>&1; echo EXIT $? >> gpurun_out/gputest_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 600 python bench.py --workload rodinia --steps 20 --warmup 5 > gpurun_out/bench_rodinia_$TAG.json 2>&1
timeout 900 python bench.py --workload batch --steps 10 --warmup 3 > gpurun_out/bench_batch_$TAG.json 2>&1
timeout 900 python bench.py --workload pelec --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_pelec_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_config3_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_config2_$TAG.csv python bench.py --workload rodinia --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_config4_$TAG.csv python tools/batch_profile.py > /dev/null 2>&1
out=gpurun_out/sanitizer_$TAG.txt
echo "# compute-sanitizer on the B200 (round 2, final session: u16 smem ingest, PDL reduce, def+rollup tiles, estimate items)" > $out
run() { echo "## $1: $2" >> $out; shift; tool=$1; shift
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -x "$@" 2>&1 | grep -E "passed|failed|SUMMARY|Error|hazard" | head -30 >> $out; }
run synccheck synccheck tests/test_gpu_parity.py -k "tiny or ragged or random_programs or wide_local or u16"
run memcheck memcheck tests/test_gpu_parity.py -k "tiny or ragged or random_programs or wide_local or skewed or u16"
run memcheck memcheck tests/test_gpu_estimate_cases.py tests/test_gpu_advice.py tests/test_gpu_fused.py
run racecheck racecheck tests/test_gpu_parity.py -k "tiny or random_programs or u16"
run racecheck racecheck tests/test_gpu_fused.py -k "tiny or rodinia"
ls -la gpurun_out/
