# Round 2, final session: the Wide exchange shape of k_ingest_part -- full GPU suite, then A/B
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_wide.log 2>&1; echo smoke $? >> gpurun_out/smoke_wide.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gt_wide.log 2>&1; echo EXIT $? >> gpurun_out/gt_wide.log
WL="large pelec" bash tools/bench_ab.sh "$@" > gpurun_out/ab_wide.txt 2>&1
