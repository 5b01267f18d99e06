for v in product build/libv_*.so; do timeout 120 python tools/variant_time.py $v 2>&1 | grep -v Warn | tail -1; done
python - <<'P'
import numpy as np, glob
ref = np.load("gpurun_out/counts_product.npy")
for f in sorted(glob.glob("gpurun_out/counts_libv*.npy")):
    print(f, "identical" if np.array_equal(np.load(f), ref) else "DIFFERENT")
P
rm -f gpurun_out/counts_*
