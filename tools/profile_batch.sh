#!/bin/bash
# One GPU session for config 4: bench line, launch list with DRAM bytes, full ncu capture of the
# step's kernels.  Outputs under gpurun_out/.
set -x
TAG=${1:-r01}
timeout 900 python bench.py --workload batch --steps 10 --warmup 3 > gpurun_out/bench_batch_$TAG.json 2> gpurun_out/bench_batch_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/batch_launches_$TAG.csv python tools/batch_profile.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ingest_seg|k_rollup_packs|k_est_rows|k_vrows|k_blame_rows" \
    -o gpurun_out/prof_batch_$TAG python tools/batch_profile.py > gpurun_out/ncu_batch_$TAG.log 2>&1
