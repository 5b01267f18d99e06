"""Seeded PC-sample streams (input generation only).

Integer alias tables are built here from a program's PC weights and reason profiles; the
records themselves come from ``csrc/gen_core.h`` compiled into ``libgpagen.so`` twice (a
host loop that feeds the CPU oracle, a CUDA kernel that fills HBM for the GPU path), so
both sides see byte-identical records.  Record k depends only on (seed, k, tables).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .programs import _PROFILES, Program, CONFIG_SEED_BASE

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgpagen.so")
STREAM_SEED_XOR = 0x9E3779B97F4A7C15


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "csrc", "gen_stream.cu")
    hdr = os.path.join(_HERE, "csrc", "gen_core.h")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(hdr)):
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
               "-shared", "-Xcompiler", "-fPIC", "-o", _LIB_PATH, src]
        subprocess.check_call(cmd)
    return _LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_instr", ctypes.c_uint32), ("n_slots", ctypes.c_uint32),
                ("n_reasons", ctypes.c_uint32), ("count_max", ctypes.c_uint32),
                ("invalid_ppm", ctypes.c_uint32), ("pc_offset", ctypes.c_uint32),
                ("pc_thresh", ctypes.c_void_p), ("pc_alias", ctypes.c_void_p),
                ("pc_profile", ctypes.c_void_p), ("slot_thresh", ctypes.c_void_p),
                ("slot_alias", ctypes.c_void_p)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.gg_generate_host.argtypes = [ctypes.POINTER(_Params), ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_void_p]
        _lib.gg_generate_device.argtypes = [ctypes.POINTER(_Params), ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    return _lib


def alias_table(weights) -> tuple[np.ndarray, np.ndarray]:
    """Vose alias table with u32 thresholds: column c keeps itself when the high draw word
    is < thresh[c], else yields alias[c]."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    p = w * n / w.sum()
    thresh = np.zeros(n, np.float64)
    alias = np.arange(n, dtype=np.int64)
    small = list(np.nonzero(p < 1.0)[0][::-1])
    large = list(np.nonzero(p >= 1.0)[0][::-1])
    p = p.copy()
    while small and large:
        s = small.pop()
        l = large.pop()
        thresh[s] = p[s]
        alias[s] = l
        p[l] = p[l] + p[s] - 1.0
        (small if p[l] < 1.0 else large).append(l)
    for rest in (small, large):
        for i in rest:
            thresh[i] = 1.0
            alias[i] = i
    t32 = np.minimum(np.floor(thresh * 2.0**32), 2.0**32 - 1).astype(np.uint64)
    t32[thresh >= 1.0] = 0xFFFFFFFF
    return t32.astype(np.uint32), alias.astype(np.uint32)


class StreamSpec:
    """Everything the generator needs; table arrays are host numpy (and optionally device)."""

    def __init__(self, prog: Program, seed: int, count_max: int = 1, invalid_ppm: int = 0):
        R = prog.n_reasons
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.n_instr = prog.n_instr
        self.n_reasons = R
        self.count_max = int(count_max)
        self.invalid_ppm = int(invalid_ppm)
        self.pc_thresh, self.pc_alias = alias_table(prog.pc_weight)
        self.pc_profile = np.ascontiguousarray(prog.pc_profile, dtype=np.uint8)
        n_prof = len(_PROFILES)
        st = np.zeros((n_prof, 2 * R), np.uint32)
        sa = np.zeros((n_prof, 2 * R), np.uint32)
        for k in range(n_prof):
            w9 = np.array(_PROFILES[k], np.float64).reshape(2, 9)
            w = np.zeros((2, R), np.float64)
            m = min(R, 9)
            w[:, :m] = w9[:, :m]
            if R > 9:
                w[:, 9:] = 1.0
            w[1, 0] = 0.0     # a latency sample always carries a stall reason
            st[k], sa[k] = alias_table(w.reshape(-1))
        self.slot_thresh, self.slot_alias = st.reshape(-1), sa.reshape(-1)
        self._dev = None

    def _params(self, ptrs) -> _Params:
        return _Params(self.seed, self.n_instr, 2 * self.n_reasons, self.n_reasons, self.count_max,
                       self.invalid_ppm, 0, *ptrs)

    def host(self, k0: int, n: int) -> np.ndarray:
        """Records [k0, k0+n) as a uint64 numpy array (8 bytes per record)."""
        lib = _load()
        out = np.empty(int(n), np.uint64)
        arrs = (self.pc_thresh, self.pc_alias, self.pc_profile, self.slot_thresh, self.slot_alias)
        prm = self._params([a.ctypes.data for a in arrs])
        lib.gg_generate_host(ctypes.byref(prm), int(k0), int(n), out.ctypes.data)
        return out

    def device(self, k0: int, n: int, out_tensor=None, stream=None):
        """Records [k0, k0+n) generated on the current CUDA device into a torch uint8 tensor
        of 8n bytes (allocated if not given)."""
        import torch
        lib = _load()
        if self._dev is None:
            self._dev = [torch.from_numpy(a.view(np.uint8).copy()).cuda() for a in (
                self.pc_thresh, self.pc_alias, self.pc_profile, self.slot_thresh, self.slot_alias)]
        if out_tensor is None:
            out_tensor = torch.empty(int(n) * 8, dtype=torch.uint8, device="cuda")
        prm = self._params([t.data_ptr() for t in self._dev])
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib.gg_generate_device(ctypes.byref(prm), int(k0), int(n), out_tensor.data_ptr(),
                                    ctypes.c_void_p(s.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"gg_generate_device failed: cuda error {rc}")
        return out_tensor


def config_stream(prog: Program, cfg: int, **kw) -> StreamSpec:
    return StreamSpec(prog, (CONFIG_SEED_BASE + cfg) ^ STREAM_SEED_XOR, **kw)
