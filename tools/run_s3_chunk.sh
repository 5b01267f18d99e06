# Round 2, final session: larger exchange chunks with 2-deep rings (k_ingest_part), config 3 A/B + parity
set -x
for v in "$@"; do GPA_LIB_PATH=$PWD/$v timeout 600 python -m pytest tests -m gpu -x -q -k "config3_large or part_skew or wide_local" > gpurun_out/gt_chunk_$(basename $v).log 2>&1; echo EXIT $? >> gpurun_out/gt_chunk_$(basename $v).log; done
WL=large bash tools/bench_ab.sh "$@" > gpurun_out/ab_chunk.txt 2>&1
