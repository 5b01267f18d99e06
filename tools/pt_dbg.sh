timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/batch_probe.py 2>&1 | grep -v Warn | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | grep -o '"value": [0-9.e+]*\|"ingest_ms": [0-9.]*\|"blame_rollup_estimate_ms": [0-9.]*'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/batch_launches.csv python tools/batch_profile.py > /dev/null 2>&1
