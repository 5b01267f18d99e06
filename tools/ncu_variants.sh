# ncu (full set) of the first config-3 ingest launch of each library variant: tools/ncu_variants.sh lib...
for v in "$@"; do
  n=$(basename $v .so)
  timeout 600 ncu --set full --clock-control none -k regex:k_ingest_part -c 1 -o gpurun_out/var_$n \
      python tools/variant_time.py $v 200000000 > gpurun_out/var_$n.log 2>&1
done
