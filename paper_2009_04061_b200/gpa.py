"""Thin Python binding of the C ABI in include/gpa.h (argument marshalling only).

Every step of GPA's hot path runs in the sm_100a kernels of libgpa_b200.so; torch is used for
device memory (the workspace is a torch uint8 tensor), streams and process groups.  There is
no CPU fallback: importing without the built library, or creating a program without a CUDA
device, raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPA_LIB_PATH") or os.path.join(_HERE, "libgpa_b200.so")   # override: tuning builds

VIEW = {
    "counts": 0, "stats": 1, "instr_al": 2, "cand": 3, "self": 4, "share": 5, "instr_blame": 6,
    "line": 7, "line_al": 8, "loop_excl": 9, "loop_excl_al": 10, "loop_incl": 11,
    "loop_incl_al": 12, "func": 13, "func_al": 14, "kernel": 15, "kernel_al": 16, "estimates": 17,
}
VARIANT = {"smem": 0, "part": 1, "l2": 2}


class GpaError(RuntimeError):
    pass


class ProgramDesc(ctypes.Structure):
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
                ("sm_count", ctypes.c_uint32), ("ratio", ctypes.c_double), ("W", ctypes.c_double),
                ("W_new", ctypes.c_double), ("f", ctypes.c_double)]


class EstimateOut(ctypes.Structure):
    _fields_ = [("speedup", ctypes.c_double), ("M", ctypes.c_double), ("eq3", ctypes.c_double),
                ("eq4", ctypes.c_double), ("T", ctypes.c_uint64), ("A", ctypes.c_uint64),
                ("best_scope", ctypes.c_int32), ("unbounded", ctypes.c_uint8),
                ("matched", ctypes.c_uint8), ("model", ctypes.c_uint8), ("pad", ctypes.c_uint8)]


class Hotspot(ctypes.Structure):
    _fields_ = [("def_pc", ctypes.c_uint32), ("use_pc", ctypes.c_uint32), ("distance", ctypes.c_uint32),
                ("item", ctypes.c_uint32), ("samples", ctypes.c_double)]


class Coverage(ctypes.Structure):
    _fields_ = [("nodes", ctypes.c_uint64), ("single_before", ctypes.c_uint64), ("single_after", ctypes.c_uint64)]


class SassDesc(ctypes.Structure):
    _fields_ = [("n_instr", ctypes.c_uint32), ("n_funcs", ctypes.c_uint32), ("n_blocks", ctypes.c_uint32)] + [
        (k, ctypes.c_void_p) for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst", "src",
                                       "wbar", "rbar", "wait")]


class SimCfg(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("schedulers", "warps_per_scheduler", "period", "trip_count",
                                               "rbar_latency", "max_cycles")] + [("seed", ctypes.c_uint64)]


class Arch(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("sm_count", "max_warps_per_sm", "max_blocks_per_sm", "regs_per_sm",
                                               "smem_per_sm", "schedulers_per_sm", "warp_size", "reg_alloc_unit")]


class Launch(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("threads_per_block", "regs_per_thread", "smem_per_block", "pad")]


# GPU limits for the occupancy model: the paper's profiled V100 and this B200
ARCH_V100 = dict(sm_count=80, max_warps_per_sm=64, max_blocks_per_sm=32, regs_per_sm=65536, smem_per_sm=98304,
                 schedulers_per_sm=4, warp_size=32, reg_alloc_unit=256)
ARCH_B200 = dict(sm_count=148, max_warps_per_sm=64, max_blocks_per_sm=32, regs_per_sm=65536, smem_per_sm=233472,
                 schedulers_per_sm=4, warp_size=32, reg_alloc_unit=256)

TOP_K_MAX = 8

EXPORTS = ["gpa_validate_program", "gpa_workspace_size", "gpa_program_create", "gpa_program_destroy",
           "gpa_reset_counts", "gpa_ingest_samples", "gpa_ingest_samples_host", "gpa_blame",
           "gpa_aggregate", "gpa_set_patterns", "gpa_estimate", "gpa_read_estimates", "gpa_get_stats",
           "gpa_view", "gpa_instr_vector", "gpa_program_info", "gpa_ingest_variant",
           "gpa_set_ingest_variant", "gpa_launch_count", "gpa_last_error", "gpa_version", "gpa_analyze",
           "gpa_ingest_segments", "gpa_advise", "gpa_read_advice", "gpa_set_launches", "gpa_slice", "gpa_simulate",
           "gpa_set_analyze_mode"]

_lib = None


def lib():
    """Load libgpa_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2009_04061_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        sig = {
            "gpa_validate_program": [vp], "gpa_workspace_size": [vp, vp],
            "gpa_program_create": [vp, vp, ctypes.c_size_t, vp, vp], "gpa_program_destroy": [vp],
            "gpa_reset_counts": [vp, vp], "gpa_ingest_samples": [vp, vp, u64, vp],
            "gpa_ingest_samples_host": [vp, vp, u64, vp], "gpa_blame": [vp, vp],
            "gpa_aggregate": [vp, vp], "gpa_set_patterns": [vp, vp, u32, vp],
            "gpa_estimate": [vp, vp], "gpa_read_estimates": [vp, vp, vp], "gpa_get_stats": [vp, vp, vp],
            "gpa_view": [vp, ctypes.c_int, vp, vp], "gpa_instr_vector": [vp, vp, vp],
            "gpa_program_info": [vp, vp], "gpa_ingest_variant": [vp, vp],
            "gpa_set_ingest_variant": [vp, ctypes.c_int], "gpa_launch_count": [vp, vp],
            "gpa_analyze": [vp, vp], "gpa_set_analyze_mode": [vp, ctypes.c_int],
            "gpa_ingest_segments": [vp, vp, u64, vp, vp, u32, u32, vp],
            "gpa_advise": [vp, u32, vp], "gpa_read_advice": [vp, vp, vp, vp, vp, vp],
            "gpa_set_launches": [vp, vp, vp, vp],
            "gpa_slice": [vp, u64, vp, vp, vp, vp, vp, vp, vp, vp],
            "gpa_simulate": [vp, vp, vp, u32, vp, u32, u64, vp, vp, vp, vp],
        }
        for name, args in sig.items():
            if os.environ.get("GPA_LIB_PATH") and not hasattr(L, name):
                continue   # an older tuning build without this call
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.gpa_last_error.restype = ctypes.c_char_p
        L.gpa_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def slice_sass(sass, stream=None):
    """Backward slicing on the GPU (gpa_slice): SASS fields + CFG (an object with the gpa_sass_desc
    arrays, e.g. gpagen.sass.Sass) -> dict of the def-use CSR (numpy): row_ptr, edge_def,
    edge_kind, edge_min_len, edge_max_len, edge_dom_k."""
    dt = {"func_begin": np.uint32, "block_begin": np.uint32, "succ_ptr": np.uint32, "succ": np.uint32,
          "guard": np.uint8, "dst": np.uint16, "src": np.uint16, "wbar": np.uint8, "rbar": np.uint8, "wait": np.uint8}
    a = {k: np.ascontiguousarray(getattr(sass, k), dtype=t) for k, t in dt.items()}
    n = int(a["guard"].shape[0])
    desc = SassDesc(n, int(a["func_begin"].shape[0] - 1), int(a["block_begin"].shape[0] - 1),
                    *[a[k].ctypes.data for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst",
                                                 "src", "wbar", "rbar", "wait")])
    row_ptr = np.zeros(n + 1, np.uint32)
    ne = ctypes.c_uint64(0)
    cap = 8 * n + 1024   # room for the usual ~2 edges per instruction: one call (a second only on overflow)
    out = None
    for _ in range(2):   # a call with too small arrays reports the edge count, then the retry fills them
        out = {"edge_def": np.zeros(max(cap, 1), np.uint32), "edge_kind": np.zeros(max(cap, 1), np.uint8),
               "edge_min_len": np.zeros(max(cap, 1), np.uint32), "edge_max_len": np.zeros(max(cap, 1), np.uint32),
               "edge_dom_k": np.zeros(max(cap, 1), np.int32)}
        rc = lib().gpa_slice(ctypes.byref(desc), cap, row_ptr.ctypes.data,
                             *[out[k].ctypes.data for k in ("edge_def", "edge_kind", "edge_min_len", "edge_max_len",
                                                            "edge_dom_k")], ctypes.byref(ne),
                             None if stream is None else ctypes.c_void_p(stream.cuda_stream))
        if rc == 0:
            break
        if rc == -7 and ne.value > cap:
            cap = int(ne.value)
            continue
        _check(rc, "gpa_slice")
    res = {k: v[: ne.value].copy() for k, v in out.items()}
    res["row_ptr"] = row_ptr
    return res


def _sass_desc(sass):
    dt = {"func_begin": np.uint32, "block_begin": np.uint32, "succ_ptr": np.uint32, "succ": np.uint32,
          "guard": np.uint8, "dst": np.uint16, "src": np.uint16, "wbar": np.uint8, "rbar": np.uint8, "wait": np.uint8}
    a = {k: np.ascontiguousarray(getattr(sass, k), dtype=t) for k, t in dt.items()}
    n = int(a["guard"].shape[0])
    desc = SassDesc(n, int(a["func_begin"].shape[0] - 1), int(a["block_begin"].shape[0] - 1),
                    *[a[k].ctypes.data for k in ("func_begin", "block_begin", "succ_ptr", "succ", "guard", "dst",
                                                 "src", "wbar", "rbar", "wait")])
    return desc, a


def simulate_sass(sass, n_sm, cap_per_sm, func=0, schedulers=4, warps_per_scheduler=4, period=4, trip_count=4,
                  rbar_latency=2, max_cycles=10_000_000, seed=1, truth=True, stream=None):
    """PC-sampling simulator on the GPU (gpa_simulate): n_sm simulated SMs running `func`.  Returns
    (records: CUDA int64 tensor [n_sm * cap_per_sm], zero-filled past each SM's count -- a zero record
    is a valid no-op sample of count 0 --, truth: CUDA int32 tensor or None, counts: numpy [n_sm])."""
    import torch
    desc, keep = _sass_desc(sass)
    cls = np.ascontiguousarray(sass.opclass, np.uint8)
    lat = np.ascontiguousarray(sass.latency, np.uint32)
    cfg = SimCfg(schedulers, warps_per_scheduler, period, trip_count, rbar_latency, max_cycles, seed)
    rec = torch.zeros(n_sm * cap_per_sm, dtype=torch.int64, device="cuda")
    tr = torch.full((n_sm * cap_per_sm,), -1, dtype=torch.int32, device="cuda") if truth else None
    counts = np.zeros(n_sm, np.uint64)
    s = torch.cuda.current_stream() if stream is None else stream
    _check(lib().gpa_simulate(ctypes.byref(desc), cls.ctypes.data, lat.ctypes.data, int(func), ctypes.byref(cfg),
                              int(n_sm), int(cap_per_sm), rec.data_ptr(), tr.data_ptr() if truth else None,
                              counts.ctypes.data, ctypes.c_void_p(s.cuda_stream)), "gpa_simulate")
    return rec, tr, counts


def _need_contiguous(t, what: str):
    """The C ABI takes a base pointer and a record count: a strided view would be read as if dense."""
    if not t.is_contiguous():
        raise GpaError(f"{what}() needs a contiguous tensor (got strides {tuple(t.stride())})")


def _check(rc: int, what: str):
    if rc != 0:
        raise GpaError(f"{what} failed ({rc}): {lib().gpa_last_error().decode()}")


_DT = {"opclass": np.uint8, "iflags": np.uint8, "latency": np.uint32, "line_id": np.uint32,
       "loop_id": np.int32, "loop_parent": np.int32, "func_begin": np.uint32,
       "kernel_func_begin": np.uint32, "kernel_grid_blocks": np.uint32, "row_ptr": np.uint32,
       "edge_def": np.uint32, "edge_kind": np.uint8, "edge_min_len": np.uint32,
       "edge_max_len": np.uint32, "edge_dom_k": np.int32}


class _Desc:
    """Host arrays of a program (kept alive) and the gpa_program_desc pointing at them."""

    def __init__(self, prog):
        self.arr = {}
        for k, dt in _DT.items():
            v = getattr(prog, k, None)
            self.arr[k] = None if v is None else np.ascontiguousarray(v, dtype=dt)
        n = int(self.arr["opclass"].shape[0])
        self.d = ProgramDesc(
            n, int(prog.n_reasons), int(prog.n_lines), int(self.arr["loop_parent"].shape[0]),
            int(self.arr["func_begin"].shape[0] - 1), int(self.arr["kernel_func_begin"].shape[0] - 1),
            *[None if self.arr[k] is None or self.arr[k].size == 0 else self.arr[k].ctypes.data for k in (
                  "opclass", "iflags", "latency", "line_id", "loop_id", "loop_parent", "func_begin",
                  "kernel_func_begin", "kernel_grid_blocks", "row_ptr", "edge_def", "edge_kind",
                  "edge_min_len", "edge_max_len", "edge_dom_k")])


def validate(prog) -> None:
    """Host-only structural validation (gpa_validate_program); raises GpaError."""
    d = _Desc(prog)
    _check(lib().gpa_validate_program(ctypes.byref(d.d)), "gpa_validate_program")


def workspace_size(prog) -> int:
    d = _Desc(prog)
    out = ctypes.c_size_t(0)
    _check(lib().gpa_workspace_size(ctypes.byref(d.d), ctypes.byref(out)), "gpa_workspace_size")
    return int(out.value)


def _pattern_struct(p) -> Pattern:
    if isinstance(p, Pattern):
        return p
    return Pattern(int(p["column_mask"]), int(p["class_mask"]), int(p["sample_class"]), int(p["model"]),
                   int(p["flag_filter"]), int(p["same_loop"]), int(p["parallel_rule"]), 0,
                   int(p["sm_count"]), float(p["ratio"]), float(p["W"]), float(p["W_new"]), float(p["f"]))


class Program:
    """One program's device workspace and handle (gpa_program_create)."""

    def __init__(self, prog, device=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise GpaError("a CUDA device is required (there is no CPU fallback)")
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self._desc = _Desc(prog)
        size = ctypes.c_size_t(0)
        _check(lib().gpa_workspace_size(ctypes.byref(self._desc.d), ctypes.byref(size)), "gpa_workspace_size")
        self.ws = torch.empty(max(int(size.value), 256), dtype=torch.uint8, device=self.device)
        self.handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().gpa_program_create(ctypes.byref(self._desc.d), self.ws.data_ptr(), self.ws.numel(),
                                            self._s(stream), ctypes.byref(self.handle)), "gpa_program_create")
        info = (ctypes.c_uint64 * 8)()
        _check(lib().gpa_program_info(self.handle, info), "gpa_program_info")
        (self.n_instr, self.n_edges, self.R, self.ncol, self.n_lines, self.n_loops, self.n_funcs,
         self.n_kernels) = (int(x) for x in info)
        self.n_patterns = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().gpa_program_destroy(h)
            except Exception:   # interpreter shutdown
                pass
            self.handle = None

    def _s(self, stream):
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    # -------------------------------------------------------------- hot path (enqueue only)
    def reset(self, stream=None):
        _check(lib().gpa_reset_counts(self.handle, self._s(stream)), "gpa_reset_counts")

    def ingest(self, samples, n=None, stream=None):
        """samples: CUDA tensor holding 8-byte records (any dtype; uint8 of 8n bytes, or int64 of n)."""
        t = samples
        if not t.is_cuda:
            raise GpaError("ingest() takes a device tensor; use ingest_host() for host memory")
        _need_contiguous(t, "ingest")
        nrec = int(t.numel() * t.element_size() // 8) if n is None else int(n)
        _check(lib().gpa_ingest_samples(self.handle, t.data_ptr(), nrec, self._s(stream)), "gpa_ingest_samples")

    def ingest_segments(self, samples, seg_begin, seg_kernel, pc_base=0, n=None, stream=None):
        """Stream grouped by kernel launch (gpa_ingest_segments): samples as in ingest();
        seg_begin: CUDA int64/uint64 tensor [S+1] of record offsets; seg_kernel: CUDA int32/uint32
        tensor [S] of kernel ids; pc_base subtracted from every pc."""
        for t in (samples, seg_begin, seg_kernel):
            if not t.is_cuda:
                raise GpaError("ingest_segments() takes device tensors")
            _need_contiguous(t, "ingest_segments")
        if seg_begin.element_size() != 8 or seg_kernel.element_size() != 4:
            raise GpaError("seg_begin must hold 8-byte and seg_kernel 4-byte integers")
        n_seg = int(seg_kernel.numel())
        if int(seg_begin.numel()) != n_seg + 1:
            raise GpaError("seg_begin needs len(seg_kernel) + 1 entries")
        nrec = int(samples.numel() * samples.element_size() // 8) if n is None else int(n)
        _check(lib().gpa_ingest_segments(self.handle, samples.data_ptr(), nrec, seg_begin.data_ptr(),
                                         seg_kernel.data_ptr(), n_seg, int(pc_base), self._s(stream)),
               "gpa_ingest_segments")

    def ingest_host(self, samples, n=None, stream=None):
        """samples: host numpy array / CPU tensor of 8-byte records (pinned memory overlaps)."""
        if hasattr(samples, "data_ptr"):
            _need_contiguous(samples, "ingest_host")
            ptr, nbytes = samples.data_ptr(), samples.numel() * samples.element_size()
        else:
            a = np.ascontiguousarray(samples)
            ptr, nbytes = a.ctypes.data, a.nbytes
        nrec = nbytes // 8 if n is None else int(n)
        _check(lib().gpa_ingest_samples_host(self.handle, ptr, nrec, self._s(stream)), "gpa_ingest_samples_host")

    def blame(self, stream=None):
        _check(lib().gpa_blame(self.handle, self._s(stream)), "gpa_blame")

    def aggregate(self, stream=None):
        _check(lib().gpa_aggregate(self.handle, self._s(stream)), "gpa_aggregate")

    def set_patterns(self, patterns, stream=None):
        arr = (Pattern * len(patterns))(*[_pattern_struct(p) for p in patterns])
        _check(lib().gpa_set_patterns(self.handle, ctypes.addressof(arr), len(patterns), self._s(stream)),
               "gpa_set_patterns")
        self.n_patterns = len(patterns)

    def estimate(self, stream=None):
        _check(lib().gpa_estimate(self.handle, self._s(stream)), "gpa_estimate")

    def analyze(self, stream=None):
        """blame + aggregate + estimate (if patterns are set): one CUDA graph replay, or one fused
        cooperative kernel for small programs (see `analyze_mode`)."""
        _check(lib().gpa_analyze(self.handle, self._s(stream)), "gpa_analyze")

    ANALYZE_MODES = {"auto": 0, "graph": 1, "fused": 2}

    @property
    def analyze_mode(self) -> str:
        return getattr(self, "_analyze_mode", "auto")

    @analyze_mode.setter
    def analyze_mode(self, mode: str):
        _check(lib().gpa_set_analyze_mode(self.handle, self.ANALYZE_MODES[mode]), "gpa_set_analyze_mode")
        self._analyze_mode = mode

    def step(self, samples, stream=None):
        """One pass of the whole hot path over one batch of device-resident records."""
        self.reset(stream)
        self.ingest(samples, stream=stream)
        self.analyze(stream)

    # -------------------------------------------------------------- results
    def read_estimates(self, stream=None):
        out = (EstimateOut * (self.n_kernels * self.n_patterns))()
        _check(lib().gpa_read_estimates(self.handle, ctypes.addressof(out), self._s(stream)), "gpa_read_estimates")
        return [[out[k * self.n_patterns + q] for q in range(self.n_patterns)] for k in range(self.n_kernels)]

    def read_estimates_array(self, stream=None):
        """Same as read_estimates() as a numpy structured array [n_kernels, n_patterns] (fields of
        gpa_estimate_out), without building Python objects per entry."""
        out = (EstimateOut * (self.n_kernels * self.n_patterns))()
        _check(lib().gpa_read_estimates(self.handle, ctypes.addressof(out), self._s(stream)), "gpa_read_estimates")
        return np.ctypeslib.as_array(out).reshape(self.n_kernels, self.n_patterns)

    def set_launches(self, launches, arch=None, stream=None):
        """launches: per kernel (threads_per_block, regs_per_thread, smem_per_block); arch: dict of
        gpa_arch fields (default ARCH_V100, the paper's GPU).  Enables parallel_rule 3 / 4."""
        a = Arch(**(arch or ARCH_V100))
        if len(launches) != self.n_kernels:
            raise GpaError(f"need {self.n_kernels} launches")
        L = (Launch * self.n_kernels)(*[Launch(int(t), int(r), int(m), 0) for t, r, m in launches])
        _check(lib().gpa_set_launches(self.handle, ctypes.addressof(L), ctypes.byref(a), self._s(stream)),
               "gpa_set_launches")

    def advise(self, top_k=5, stream=None):
        """Hotspots, ranking and single dependency coverage (gpa_advise) of the current estimates."""
        self._top_k = int(top_k)
        _check(lib().gpa_advise(self.handle, self._top_k, self._s(stream)), "gpa_advise")

    def read_advice(self, stream=None):
        """dict: 'hotspots' structured [K, Q, top_k] (first n valid), 'n' u32 [K, Q],
        'rank' u32 [K, Q] (pattern index per rank), 'coverage' structured [K]."""
        K, Q, T = self.n_kernels, self.n_patterns, getattr(self, "_top_k", 0)
        hot = (Hotspot * max(1, K * Q * T))()
        cov = (Coverage * K)()
        n = np.zeros((K, Q), np.uint32)
        rank = np.zeros((K, Q), np.uint32)
        _check(lib().gpa_read_advice(self.handle, ctypes.addressof(hot), n.ctypes.data, rank.ctypes.data,
                                     ctypes.addressof(cov), self._s(stream)), "gpa_read_advice")
        return {"hotspots": np.ctypeslib.as_array(hot)[:K * Q * T].reshape(K, Q, T), "n": n, "rank": rank,
                "coverage": np.ctypeslib.as_array(cov).reshape(K)}

    def stats(self, stream=None):
        out = (ctypes.c_uint64 * 4)()
        _check(lib().gpa_get_stats(self.handle, out, self._s(stream)), "gpa_get_stats")
        return [int(x) for x in out]

    def reduce_view(self):
        """int64 view (no copy) of the count table followed by the 4 stats words: the one buffer a
        data-parallel step all-reduces (they are contiguous in the workspace by construction)."""
        torch = self.torch
        offs = []
        for name in ("counts", "stats"):
            off, nb = ctypes.c_uint64(0), ctypes.c_uint64(0)
            _check(lib().gpa_view(self.handle, VIEW[name], ctypes.byref(off), ctypes.byref(nb)), "gpa_view")
            offs.append((off.value, nb.value))
        (c0, cn), (s0, sn) = offs
        if s0 != c0 + cn:
            raise RuntimeError("count table and stats are not contiguous in the workspace")
        return self.ws[c0: s0 + sn].view(torch.int64)

    def view(self, name):
        """torch view (no copy) of a device result inside the workspace."""
        torch = self.torch
        off, nb = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(lib().gpa_view(self.handle, VIEW[name], ctypes.byref(off), ctypes.byref(nb)), "gpa_view")
        raw = self.ws[off.value: off.value + nb.value]
        shapes = {
            "counts": (torch.int64, (self.n_instr, 2, self.R)), "stats": (torch.int64, (4,)),
            "instr_al": (torch.int64, (self.n_instr, 2)), "cand": (torch.uint8, (self.n_edges,)),
            "self": (torch.uint8, (self.n_instr,)), "share": (torch.float64, (self.n_edges, 3)),
            "instr_blame": (torch.float64, (self.n_instr, 4, 2)),
            "line": (torch.float64, (self.n_lines, self.ncol, 2)), "line_al": (torch.int64, (self.n_lines, 2)),
            "loop_excl": (torch.float64, (self.n_loops, self.ncol, 2)),
            "loop_excl_al": (torch.int64, (self.n_loops, 2)),
            "loop_incl": (torch.float64, (self.n_loops, self.ncol, 2)),
            "loop_incl_al": (torch.int64, (self.n_loops, 2)),
            "func": (torch.float64, (self.n_funcs, self.ncol, 2)), "func_al": (torch.int64, (self.n_funcs, 2)),
            "kernel": (torch.float64, (self.n_kernels, self.ncol, 2)),
            "kernel_al": (torch.int64, (self.n_kernels, 2)),
        }
        if name == "estimates":
            return raw
        dt, shape = shapes[name]
        return raw.view(dt).view(shape)

    def instr_vector(self, stream=None):
        torch = self.torch
        out = torch.empty((self.n_instr, self.ncol, 2), dtype=torch.float64, device=self.device)
        _check(lib().gpa_instr_vector(self.handle, out.data_ptr(), self._s(stream)), "gpa_instr_vector")
        return out

    @property
    def variant(self) -> str:
        v = ctypes.c_int(0)
        _check(lib().gpa_ingest_variant(self.handle, ctypes.byref(v)), "gpa_ingest_variant")
        return {b: a for a, b in VARIANT.items()}[v.value]

    @variant.setter
    def variant(self, name: str):
        _check(lib().gpa_set_ingest_variant(self.handle, VARIANT[name]), "gpa_set_ingest_variant")

    @property
    def launches(self) -> int:
        v = ctypes.c_uint64(0)
        _check(lib().gpa_launch_count(self.handle, ctypes.byref(v)), "gpa_launch_count")
        return int(v.value)
