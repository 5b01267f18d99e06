# A/B timing of ingest variants (config 3, 1e9 records): product vs build/lib*.so given as args,
# interleaved passes; every variant's count table compared with the product's
for i in 1 2 3; do
  python tools/variant_time.py product 1000000000
  for v in "$@"; do python tools/variant_time.py $v 1000000000; done
done
python - "$@" <<'PY'
import sys, numpy as np, os
a=np.load("gpurun_out/counts3_product.npy")
for v in sys.argv[1:]:
    b=np.load("gpurun_out/counts3_"+os.path.basename(v)+".npy"); print(v, "equal", np.array_equal(a,b))
PY
