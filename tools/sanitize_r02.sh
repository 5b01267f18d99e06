# compute-sanitizer pass (round 2): synccheck / memcheck / racecheck on the GPU tests' small cases
out=gpurun_out/sanitizer_r02.txt
echo "# compute-sanitizer on the B200 (round 2)" > $out
run() { echo "## $1: $2" >> $out; shift; tool=$1; shift
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -x "$@" 2>&1 | grep -E "passed|failed|SUMMARY|Error|hazard" | head -30 >> $out; }
run synccheck synccheck tests/test_gpu_parity.py -k "tiny or ragged or random_programs or wide_local"
run synccheck synccheck tests/test_gpu_estimate_cases.py tests/test_gpu_batch.py tests/test_gpu_slicing.py -k "not config4 and not nccl"
run memcheck memcheck tests/test_gpu_parity.py -k "tiny or ragged or random_programs or wide_local or skewed"
run memcheck memcheck tests/test_gpu_estimate_cases.py tests/test_gpu_advice.py tests/test_gpu_slicing.py tests/test_gpu_simulator.py
run racecheck racecheck tests/test_gpu_parity.py -k "tiny or random_programs"
run memcheck memcheck tests/test_gpu_fused.py tests/test_gpu_fuzz.py -k "not config3"
run racecheck racecheck tests/test_gpu_fused.py -k "tiny or rodinia"
cat $out
