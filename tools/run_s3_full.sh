# Round 2, third session: the full GPU suite and smoke on the product library, then A/B steps
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo smoke $? >> gpurun_out/smoke_full.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gt_full.log 2>&1; echo EXIT $? >> gpurun_out/gt_full.log
WL="${WL:-batch large rodinia}" bash tools/bench_ab.sh "$@" > gpurun_out/ab.txt 2>&1
