for rep in 1 2; do
for v in product build/libv_*.so; do timeout 120 python tools/variant_time.py $v 2>&1 | grep -v Warn | tail -1; done
done
rm -f gpurun_out/counts_*
for v in build/libv_el.so build/libv_plain_el.so; do
GPA_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ingest_part -c 1 python tools/variant_time.py $v 2>&1 | grep -E "dram__|gpu__time"
done
