# A/B of the analysis (configs 2,3,4): product vs build/lib*.so given as args, two passes, estimates compared
for i in 1 2; do
  for v in product "$@"; do timeout 300 python tools/analyze_time.py $v 2,3,4 graph; done
done
python - "$@" <<'PY'
import sys, os, numpy as np
for cfg in (2, 3, 4):
    a = np.load(f"gpurun_out/est_{cfg}_product_graph.npy")
    for v in sys.argv[1:]:
        b = np.load(f"gpurun_out/est_{cfg}_{os.path.basename(v)}_graph.npy")
        print(cfg, v, "identical", bool(np.array_equal(a, b)))
PY
