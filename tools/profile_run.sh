#!/bin/bash
# One GPU session: full bench line, launch list (ncu, timing only), full ncu capture of the
# ingest kernel at the bench size, clocks.  Outputs under gpurun_out/.
set -x
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest -c 1 \
    -o gpurun_out/prof_ingest_$TAG python bench.py --profile > gpurun_out/ncu_ingest_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_ingest -c 2 \
    -o gpurun_out/prof_ingest_rodinia_$TAG python bench.py --profile --workload rodinia > /dev/null 2>&1
ls -la gpurun_out/
