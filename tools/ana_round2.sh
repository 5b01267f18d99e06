# round-2 A/B of the analysis graph (configs 2, 3, 4) and GPU parity of the analysis kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in product "$@"; do python tools/analyze_time.py $v 2,3,4; done
python - "$@" <<'PY'
import sys, os, numpy as np
for cfg in (2, 3, 4):
    a = np.load(f"gpurun_out/est_{cfg}_product.npy")
    for v in sys.argv[1:]:
        b = np.load(f"gpurun_out/est_{cfg}_{os.path.basename(v)}.npy")
        print(cfg, v, "max rel diff", float(np.nanmax(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))))
PY
