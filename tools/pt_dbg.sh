timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_advice.py -x -q 2>&1 | tail -1
for v in "" build/libv_eg8.so build/libv_eg2.so; do echo "lib=$v"; GPA_LIB_PATH=$v timeout 600 python tools/batch_probe.py 2>&1 | grep -v Warn | grep "^reset " | tail -1; done
