"""Build a GPA_PART_TIMING variant of the library, run the config-3 ingest once, print phase cycles."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import gpagen
from paper_2009_04061_b200 import gpa as G
lib_path = os.path.join(ROOT, "build", "libgpa_timing.so")
G.LIB_PATH = lib_path
lib = G.lib()
prog = gpagen.config_program(3)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
recs = gpagen.config_stream(prog, 3).device(0, n)
P = G.Program(prog)
for it in range(2):
    P.reset(); P.ingest(recs); torch.cuda.synchronize()
# read the device symbol via cudaMemcpyFromSymbol through a tiny helper: use cuda-python-free route
cudart = ctypes.CDLL("libcudart.so") if False else None
names = ["dec:wait_buf", "dec:wait_ring", "dec:decode", "ctl:wait_decoded", "ctl:spin_cons+tma", "ctl:wait_store",
         "ctl:publish", "ctl:recycle", "con:fetch(spin)", "con:wait_inbox", "con:process", "con:barrier"]
buf = (ctypes.c_ulonglong * 16)()
lib.gpa_debug_read_timing.argtypes = [ctypes.c_void_p]
lib.gpa_debug_read_timing(buf)
tot_dec = sum(buf[i] for i in range(3)) or 1
tot_ctl = sum(buf[i] for i in range(3, 8)) or 1
tot_con = sum(buf[i] for i in range(8, 12)) or 1
for i, nm in enumerate(names):
    grp = tot_dec if i < 3 else tot_ctl if i < 8 else tot_con
    print(f"{nm:22s} {buf[i]/1e9:10.3f} Gcyc  {100*buf[i]/grp:5.1f}% of role")
