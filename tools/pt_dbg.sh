timeout 300 compute-sanitizer --tool memcheck --show-backtrace no python tools/part_debug.py 3000000 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for v in product product; do timeout 120 python tools/variant_time.py $v 2>&1 | grep -v Warn | tail -1; done
rm -f gpurun_out/counts_*
