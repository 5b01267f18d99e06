"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``libgpa_oracle.so`` (plain single-threaded C of GPA's definitions,
see gpa_oracle.h).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgpa_oracle.so")

P_U8 = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gpa_oracle.c")
    hdr = os.path.join(_HERE, "gpa_oracle.h")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o",
                               LIB_PATH, src, "-lm"])
    return LIB_PATH


class _Prog(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in
                ("n_instr", "n_reasons", "n_lines", "n_loops", "n_funcs", "n_kernels")] + [
        (k, ctypes.c_void_p) for k in (
            "opclass", "iflags", "latency", "line_id", "loop_id", "loop_parent", "func_begin",
            "kernel_func_begin", "kernel_grid_blocks", "row_ptr", "edge_def", "edge_kind",
            "edge_min_len", "edge_max_len", "edge_dom_k")]


class Pattern(ctypes.Structure):
    _fields_ = [("column_mask", ctypes.c_uint32), ("class_mask", ctypes.c_uint16),
                ("sample_class", ctypes.c_uint8), ("model", ctypes.c_uint8),
                ("flag_filter", ctypes.c_uint8), ("same_loop", ctypes.c_uint8),
                ("parallel_rule", ctypes.c_uint8), ("pad", ctypes.c_uint8),
                ("sm_count", ctypes.c_uint32),
                ("ratio", ctypes.c_double), ("W", ctypes.c_double), ("W_new", ctypes.c_double),
                ("f", ctypes.c_double)]


class Estimate(ctypes.Structure):
    _fields_ = [("speedup", ctypes.c_double), ("M", ctypes.c_double), ("eq3", ctypes.c_double),
                ("eq4", ctypes.c_double), ("T", ctypes.c_uint64), ("A", ctypes.c_uint64),
                ("best_scope", ctypes.c_int32), ("unbounded", ctypes.c_uint8),
                ("matched", ctypes.c_uint8), ("model", ctypes.c_uint8), ("pad", ctypes.c_uint8)]


class Arch(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("sm_count", "max_warps_per_sm", "max_blocks_per_sm", "regs_per_sm",
                                               "smem_per_sm", "schedulers_per_sm", "warp_size", "reg_alloc_unit")]


class Launch(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("threads_per_block", "regs_per_thread", "smem_per_block", "pad")]


class Occ(ctypes.Structure):
    _fields_ = [("W", ctypes.c_double), ("W_new_block", ctypes.c_double), ("W_new_thread", ctypes.c_double),
                ("blocks_per_sm", ctypes.c_uint32), ("limiter", ctypes.c_uint32),
                ("match_block", ctypes.c_uint32), ("match_thread", ctypes.c_uint32)]


class Hotspot(ctypes.Structure):
    _fields_ = [("def_pc", ctypes.c_uint32), ("use_pc", ctypes.c_uint32), ("distance", ctypes.c_uint32),
                ("item", ctypes.c_uint32), ("samples", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        L.or_histogram.argtypes = [vp, vp, ctypes.c_uint64, vp, vp]
        L.or_blame.argtypes = [vp, vp, vp, vp, vp, vp]
        L.or_rollup.argtypes = [vp] * 13
        L.or_estimate_all.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_uint32, vp]
        L.or_estimate_all_occ.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_uint32, vp, vp]
        L.or_occupancy.argtypes = [vp, vp, vp, ctypes.c_uint32, vp]
        L.or_slice.argtypes = [vp, ctypes.c_uint64, vp, vp, vp, vp, vp, vp]
        L.or_slice.restype = ctypes.c_int64
        L.or_simulate.argtypes = [vp, vp, vp, ctypes.c_uint32, vp, ctypes.c_uint32, ctypes.c_uint64, vp, vp]
        L.or_simulate.restype = ctypes.c_int64
        L.or_hotspots.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_uint32, ctypes.c_uint32, vp, vp]
        L.or_rank.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, vp]
        L.or_coverage.argtypes = [vp, vp, vp, vp]
        for f in ("or_eq2", "or_eq4", "or_eq5", "or_eq10"):
            getattr(L, f).restype = ctypes.c_double
        L.or_eq2.argtypes = [ctypes.c_double] * 2
        L.or_eq4.argtypes = [ctypes.c_double] * 3
        L.or_eq5.argtypes = [ctypes.c_double] * 3
        L.or_eq10.argtypes = [ctypes.c_double] * 4
        L.or_ncol.argtypes = [ctypes.c_uint32]
        L.or_ncol.restype = ctypes.c_uint32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleProgram:
    """Keeps the numpy arrays alive and exposes the or_program struct."""

    _DT = {"opclass": np.uint8, "iflags": np.uint8, "latency": np.uint32, "line_id": np.uint32,
           "loop_id": np.int32, "loop_parent": np.int32, "func_begin": np.uint32,
           "kernel_func_begin": np.uint32, "kernel_grid_blocks": np.uint32, "row_ptr": np.uint32,
           "edge_def": np.uint32, "edge_kind": np.uint8, "edge_min_len": np.uint32,
           "edge_max_len": np.uint32, "edge_dom_k": np.int32}

    def __init__(self, prog):
        self.arr = {k: np.ascontiguousarray(getattr(prog, k), dtype=dt) for k, dt in self._DT.items()}
        self.n_instr = int(self.arr["opclass"].shape[0])
        self.R = int(prog.n_reasons)
        self.n_lines = int(prog.n_lines)
        self.n_loops = int(self.arr["loop_parent"].shape[0])
        self.n_funcs = int(self.arr["func_begin"].shape[0] - 1)
        self.n_kernels = int(self.arr["kernel_func_begin"].shape[0] - 1)
        self.E = int(self.arr["row_ptr"][-1])
        self.ncol = int(lib().or_ncol(self.R))
        self.s = _Prog(self.n_instr, self.R, self.n_lines, self.n_loops, self.n_funcs,
                       self.n_kernels, *[_ptr(self.arr[k]) for k in (
                           "opclass", "iflags", "latency", "line_id", "loop_id", "loop_parent",
                           "func_begin", "kernel_func_begin", "kernel_grid_blocks", "row_ptr",
                           "edge_def", "edge_kind", "edge_min_len", "edge_max_len", "edge_dom_k")])

    @property
    def ref(self):
        return ctypes.byref(self.s)

    # --- step 1
    def new_counts(self) -> np.ndarray:
        return np.zeros((self.n_instr, 2, self.R), np.uint64)

    def histogram(self, records: np.ndarray, C: np.ndarray | None = None, stats=None):
        """records: uint64 array (one 8-byte record each). Accumulates into C / stats."""
        rec = np.ascontiguousarray(records).view(np.uint8)
        if C is None:
            C = self.new_counts()
        if stats is None:
            stats = np.zeros(3, np.uint64)
        lib().or_histogram(self.ref, rec.ctypes.data, rec.size // 8, C.ctypes.data, stats.ctypes.data)
        return C, stats

    # --- steps 2-6
    def blame(self, C: np.ndarray):
        cand = np.zeros(self.E, np.uint8)
        selff = np.zeros(self.n_instr, np.uint8)
        share = np.zeros((self.E, 3), np.float64)
        V = np.zeros((self.n_instr, self.ncol, 2), np.float64)
        lib().or_blame(self.ref, C.ctypes.data, cand.ctypes.data, selff.ctypes.data,
                       share.ctypes.data, V.ctypes.data)
        return {"cand": cand, "self": selff, "share": share, "V": V}

    # --- step 7
    def rollup(self, C: np.ndarray, V: np.ndarray):
        nc = self.ncol
        out = {
            "line_v": np.zeros((self.n_lines, nc, 2)), "line_al": np.zeros((self.n_lines, 2), np.uint64),
            "loop_excl_v": np.zeros((self.n_loops, nc, 2)), "loop_excl_al": np.zeros((self.n_loops, 2), np.uint64),
            "loop_incl_v": np.zeros((self.n_loops, nc, 2)), "loop_incl_al": np.zeros((self.n_loops, 2), np.uint64),
            "func_v": np.zeros((self.n_funcs, nc, 2)), "func_al": np.zeros((self.n_funcs, 2), np.uint64),
            "kern_v": np.zeros((self.n_kernels, nc, 2)), "kern_al": np.zeros((self.n_kernels, 2), np.uint64),
        }
        keys = ["line_v", "line_al", "loop_excl_v", "loop_excl_al", "loop_incl_v", "loop_incl_al",
                "func_v", "func_al", "kern_v", "kern_al"]
        lib().or_rollup(self.ref, C.ctypes.data, V.ctypes.data, *[_ptr(out[k]) for k in keys])
        return out

    # --- step 8
    def estimate(self, C, blame, patterns, occ=None):
        """occ: ctypes array of Occ per kernel (occupancy(...)) for parallel_rule 3 / 4, or None."""
        pats = (Pattern * len(patterns))(*patterns)
        out = (Estimate * (self.n_kernels * len(patterns)))()
        lib().or_estimate_all_occ(self.ref, C.ctypes.data, blame["cand"].ctypes.data,
                                  blame["self"].ctypes.data, blame["share"].ctypes.data,
                                  ctypes.addressof(pats), len(patterns),
                                  None if occ is None else ctypes.addressof(occ), ctypes.addressof(out))
        return [[out[k * len(patterns) + q] for q in range(len(patterns))]
                for k in range(self.n_kernels)]

    def run_all(self, records, patterns=None):
        C, stats = self.histogram(records)
        b = self.blame(C)
        r = self.rollup(C, b["V"])
        est = self.estimate(C, b, patterns) if patterns else None
        return {"C": C, "stats": stats, **b, **r, "est": est}


    # --- after the path: advice (hotspots, ranking, single dependency coverage)
    def hotspots(self, C, blame, patterns, top_k):
        """(list [K][Q] of lists of Hotspot) for the pattern list."""
        K, Q = self.n_kernels, len(patterns)
        pats = (Pattern * Q)(*patterns)
        out = (Hotspot * (K * Q * top_k))()
        n_out = np.zeros(K * Q, np.uint32)
        lib().or_hotspots(self.ref, C.ctypes.data, blame["cand"].ctypes.data, blame["self"].ctypes.data,
                          blame["share"].ctypes.data, ctypes.addressof(pats), Q, top_k,
                          ctypes.addressof(out), n_out.ctypes.data)
        return [[[out[(k * Q + q) * top_k + t] for t in range(int(n_out[k * Q + q]))] for q in range(Q)]
                for k in range(K)]

    def coverage(self, C, cand):
        """uint64 [K, 3]: nodes, single-dependency nodes before pruning, after pruning."""
        out = np.zeros((self.n_kernels, 3), np.uint64)
        lib().or_coverage(self.ref, C.ctypes.data, cand.ctypes.data, out.ctypes.data)
        return out


def eq2(T, M):
    return lib().or_eq2(T, M)


def eq4(T, A, ML):
    return lib().or_eq4(T, A, ML)


def eq5(T, A_nested, ML):
    return lib().or_eq5(T, A_nested, ML)


def eq10(W, W_new, R_I, f):
    return lib().or_eq10(W, W_new, R_I, f)

def rank(est):
    """est: list [K][Q] of Estimate -> uint32 [K, Q] pattern order by speedup (or_rank)."""
    K, Q = len(est), len(est[0]) if est else 0
    flat = (Estimate * (K * Q))(*[e for row in est for e in row])
    order = np.zeros((K, Q), np.uint32)
    lib().or_rank(ctypes.addressof(flat), K, Q, order.ctypes.data)
    return order


def occupancy(arch, launches, grid_blocks):
    """arch: Arch; launches: list of Launch (one per kernel); grid_blocks: sequence -> ctypes Occ array."""
    K = len(launches)
    L = (Launch * K)(*launches)
    g = np.ascontiguousarray(grid_blocks, dtype=np.uint32)
    out = (Occ * K)()
    lib().or_occupancy(ctypes.byref(arch), ctypes.addressof(L), g.ctypes.data, K, ctypes.addressof(out))
    return out


class _Sass(ctypes.Structure):
    _fields_ = [("n_instr", ctypes.c_uint32), ("n_funcs", ctypes.c_uint32), ("n_blocks", ctypes.c_uint32)] + [
        (k, ctypes.c_void_p) for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst", "src",
                                       "wbar", "rbar", "wait")]


def slice_program(sass):
    """Backward slicing (or_slice) of a SASS description (object with the or_sass arrays) ->
    dict of the def-use CSR: row_ptr, edge_def, edge_kind, edge_min_len, edge_max_len, edge_dom_k."""
    dt = {"func_begin": np.uint32, "block_begin": np.uint32, "succ_ptr": np.uint32, "succ": np.uint32,
          "guard": np.uint8, "dst": np.uint16, "src": np.uint16, "wbar": np.uint8, "rbar": np.uint8, "wait": np.uint8}
    a = {k: np.ascontiguousarray(getattr(sass, k), dtype=t) for k, t in dt.items()}
    n = int(a["guard"].shape[0])
    st = _Sass(n, int(a["func_begin"].shape[0] - 1), int(a["block_begin"].shape[0] - 1),
               *[a[k].ctypes.data for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst", "src",
                                            "wbar", "rbar", "wait")])
    cap = 64 * max(n, 1)
    row_ptr = np.zeros(n + 1, np.uint32)
    out = {"edge_def": np.zeros(cap, np.uint32), "edge_kind": np.zeros(cap, np.uint8),
           "edge_min_len": np.zeros(cap, np.uint32), "edge_max_len": np.zeros(cap, np.uint32),
           "edge_dom_k": np.zeros(cap, np.int32)}
    E = lib().or_slice(ctypes.byref(st), cap, row_ptr.ctypes.data, *[out[k].ctypes.data for k in (
        "edge_def", "edge_kind", "edge_min_len", "edge_max_len", "edge_dom_k")])
    if E < 0:
        raise RuntimeError(f"or_slice failed ({E})")
    res = {k: v[:E].copy() for k, v in out.items()}
    res["row_ptr"] = row_ptr
    return res


class SimCfg(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("schedulers", "warps_per_scheduler", "period", "trip_count",
                                               "rbar_latency", "max_cycles")] + [("seed", ctypes.c_uint64)]


def simulate(sass, cfg, sm=0, func=0, cap=1 << 22):
    """or_simulate: (records uint64 [n], truth int32 [n]) of SM `sm` running function `func`."""
    dt = {"func_begin": np.uint32, "block_begin": np.uint32, "succ_ptr": np.uint32, "succ": np.uint32,
          "guard": np.uint8, "dst": np.uint16, "src": np.uint16, "wbar": np.uint8, "rbar": np.uint8, "wait": np.uint8}
    a = {k: np.ascontiguousarray(getattr(sass, k), dtype=t) for k, t in dt.items()}
    n = int(a["guard"].shape[0])
    st = _Sass(n, int(a["func_begin"].shape[0] - 1), int(a["block_begin"].shape[0] - 1),
               *[a[k].ctypes.data for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst", "src",
                                            "wbar", "rbar", "wait")])
    cls = np.ascontiguousarray(sass.opclass, np.uint8)
    lat = np.ascontiguousarray(sass.latency, np.uint32)
    rec = np.zeros(cap, np.uint64)
    truth = np.zeros(cap, np.int32)
    m = lib().or_simulate(ctypes.byref(st), cls.ctypes.data, lat.ctypes.data, func, ctypes.byref(cfg), sm, cap,
                          rec.ctypes.data, truth.ctypes.data)
    if m < 0:
        raise RuntimeError(f"or_simulate failed ({m})")
    return rec[:m].copy(), truth[:m].copy()
