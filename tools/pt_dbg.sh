for v in "" build/libv_eg12.so build/libv_eg16.so build/libv_eg4.so build/libv_rm16.so build/libv_rm4.so; do
  echo "lib=$v"; GPA_LIB_PATH=$v timeout 600 python tools/batch_probe.py 2>&1 | grep -v Warn | grep "^reset " | tail -2
done
