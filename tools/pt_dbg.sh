timeout 300 compute-sanitizer --tool memcheck --show-backtrace no python tools/part_debug.py 3000000 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | grep -o '"value": [0-9.e+]*\|"ingest_ms": [0-9.]*\|"frac": [0-9.]*\|"blame_rollup_estimate_ms": [0-9.]*'
timeout 60 python -u tools/part_timing.py 1000000000 2>&1 | grep -v Warn | tail -6
