"""Build-variant probe: run the config-3 ingest with the GPA_PART_TIMING library (build/libgpa_timing.so,
built by paper_2009_04061_b200.build.build_variant) and print the per-role phase cycles.
Each thread accumulates its phases in registers and adds them to the global timers once."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import gpagen
from paper_2009_04061_b200 import gpa as G

G.LIB_PATH = os.path.join(ROOT, os.environ.get("PT_LIB", "build/libgpa_timing.so"))
lib = G.lib()
prog = gpagen.config_program(3)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
recs = gpagen.config_stream(prog, 3).device(0, n)
P = G.Program(prog)
buf = (ctypes.c_ulonglong * 16)()
lib.gpa_debug_read_timing.argtypes = [ctypes.c_void_p]
for it in range(2):      # the second pass is the measured one
    lib.gpa_debug_read_timing(buf)
    before = list(buf)
    P.reset(); P.ingest(recs); torch.cuda.synchronize()
    lib.gpa_debug_read_timing(buf)
delta = [buf[i] - before[i] for i in range(16)]
roles = {
    "decoders (per warp)": ([0, 2], ["load+wait_buf", "decode"]),
    "control": ([3, 4, 5], ["wait_decoded", "spin_cons", "store+wait_group"]),
    "publisher": ([14, 15, 7], ["wait_stored", "publish", "recycle"]),
    "loader": ([12, 13], ["wait_inbox_full(+spin_prod)", "wait_processors"]),
    "processors (per warp)": ([9, 10, 11], ["wait_full", "process", "flush"]),
}
for role, (slots, names) in roles.items():
    tot = sum(delta[s] for s in slots) or 1
    print(role + ": " + ", ".join(f"{nm} {100 * delta[s] / tot:.1f}%" for s, nm in zip(slots, names))
          + f"  (total {tot / 1e9:.2f} Gcyc)")
