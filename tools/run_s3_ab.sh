set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or fuzz or estimate or batch or fused or advice or fullsize" > gpurun_out/gt2.log 2>&1; echo EXIT $? >> gpurun_out/gt2.log
WL="batch large rodinia" bash tools/bench_ab.sh build/libbe0.so build/libg4.so build/libg16.so > gpurun_out/ab2.txt 2>&1
