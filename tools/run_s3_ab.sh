# Round 2, third session: GPU tests of the product library, then whole-step A/B against variants
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or fuzz or estimate or batch or fused or advice or fullsize" > gpurun_out/gt_ab.log 2>&1; echo EXIT $? >> gpurun_out/gt_ab.log
WL="${WL:-batch large rodinia}" bash tools/bench_ab.sh "$@" > gpurun_out/ab.txt 2>&1
