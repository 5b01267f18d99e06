for v in "" build/libv_*.so; do echo "lib=$v"; GPA_LIB_PATH=$v timeout 600 python tools/batch_probe.py 2>&1 | grep -v Warn | grep "^reset " | tail -1; done
