# Round-2 GPU session: bench lines (config 3 default, reference arm, rodinia, batch, pelec), launch
# lists with DRAM bytes, one full ncu capture of the ingest kernel.  Outputs under gpurun_out/.
set -x
TAG=r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 600 python bench.py --workload rodinia --steps 20 --warmup 5 > gpurun_out/bench_rodinia_$TAG.json 2>&1
timeout 900 python bench.py --workload batch --steps 10 --warmup 3 > gpurun_out/bench_batch_$TAG.json 2>&1
timeout 900 python bench.py --workload pelec --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_pelec_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_rodinia_$TAG.csv python bench.py --workload rodinia --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/batch_launches_$TAG.csv python tools/batch_profile.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_part -c 1 \
    -o gpurun_out/prof_ingest_$TAG python bench.py --profile > gpurun_out/ncu_ingest_$TAG.log 2>&1
ls -la gpurun_out/
