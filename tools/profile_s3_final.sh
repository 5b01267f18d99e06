#!/bin/bash
# Round 2, final session: smoke, the full GPU suite, bench lines for every workload and the
# reference arm, ncu launch lists (config 3, config 2, config 4), ncu --set full of the ingest kernel
# (compute-sanitizer is closed on the pool).
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_part -c 1 \
    -o gpurun_out/prof_ingest_$TAG python bench.py --profile > gpurun_out/ncu_ingest_$TAG.log 2>&1
ls -la gpurun_out/
