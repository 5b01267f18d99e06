# round-2 A/B timing of ingest variants (config 3, 1e9 records): product vs build/lib*.so given as args
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
  python tools/variant_time.py product 1000000000
  for v in "$@"; do python tools/variant_time.py $v 1000000000; done
done
python - "$@" <<'PY'
import sys, numpy as np, os
a=np.load("gpurun_out/counts_product.npy")
for v in sys.argv[1:]:
    b=np.load("gpurun_out/counts_"+os.path.basename(v)+".npy"); print(v, "equal", np.array_equal(a,b))
PY
