# A/B of whole bench steps: product vs GPA_LIB_PATH=build/lib*.so, for the workloads in $WL (default batch)
WL=${WL:-batch}
for i in 1 2; do
  for v in product "$@"; do
    for w in $WL; do
      if [ $v = product ]; then L=""; else L="GPA_LIB_PATH=$PWD/$v"; fi
      env $L timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '$w', round(d['ms_per_step'],4), 'ingest', round(r['ingest_ms'],4), 'analysis', round(r['blame_rollup_estimate_ms'],4))"
    done
  done
done
