# Round 2, third session: u16 table of the partitioned ingest (14/15-bit local bins)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "part or wide or skew or fullsize or u16" > gpurun_out/gt_pelec.log 2>&1; echo EXIT $? >> gpurun_out/gt_pelec.log
for i in 1 2; do for v in product "$@"; do
  if [ $v = product ]; then L=""; else L="GPA_LIB_PATH=$PWD/$v"; fi
  for w in pelec large; do
  env $L timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '$w', round(d['ms_per_step'],4), 'ingest', round(r['ingest_ms'],4), 'frac', round(r['frac'],4))" >> gpurun_out/ab_pelec.txt
  done
done; done
