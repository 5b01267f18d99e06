# A/B timing of the config-2 (smem variant) ingest: product vs build/lib*.so given as args
for i in 1 2 3; do
  python tools/variant_time.py product 10000000 2
  for v in "$@"; do python tools/variant_time.py $v 10000000 2; done
done
python - "$@" <<'PY'
import sys, numpy as np, os
a=np.load("gpurun_out/counts2_product.npy")
for v in sys.argv[1:]:
    b=np.load("gpurun_out/counts2_"+os.path.basename(v)+".npy"); print(v, "equal", np.array_equal(a,b))
PY
