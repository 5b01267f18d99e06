for v in "" build/libv_*.so; do GPA_LIB_PATH=$v timeout 300 python tools/seg_time.py 2>&1 | grep -v Warn | tail -1; done
