for v in product build/libv_*.so; do timeout 120 python tools/variant_time.py $v 2>&1 | grep -v Warn | tail -1; done
rm -f gpurun_out/counts_*
