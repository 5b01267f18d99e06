"""Shared test helpers: run the CUDA path and the oracle on the same seeded inputs."""
import numpy as np

import oracle
from gpagen.patterns import table2

PATTERN_KEYS = ("column_mask", "class_mask", "sample_class", "model", "flag_filter", "same_loop",
                "parallel_rule")


def oracle_pattern(d):
    return oracle.Pattern(*[d[k] for k in PATTERN_KEYS], 0, d["sm_count"], d["ratio"], d["W"],
                          d["W_new"], d["f"])


def run_oracle(prog, records, patterns=None, chunk=None):
    patterns = table2(prog.n_reasons) if patterns is None else patterns
    op = oracle.OracleProgram(prog)
    if chunk is None:
        C, stats = op.histogram(records)
    else:
        C, stats = None, None
        for k in range(0, len(records), chunk):
            C, stats = op.histogram(records[k:k + chunk], C, stats)
    b = op.blame(C)
    r = op.rollup(C, b["V"])
    est = op.estimate(C, b, [oracle_pattern(p) for p in patterns])
    return {"C": C, "stats": stats, **b, **r, "est": est}


def run_gpu(prog, records, patterns=None, variant=None, host=False, offset_records=0, segments=None,
            analyze=None):
    """records: numpy uint64 array.  offset_records: place the stream at an 8-byte (not 16-byte)
    aligned address to exercise the unaligned head.  segments: (seg_begin, seg_kernel, pc_base)
    to ingest through gpa_ingest_segments (records grouped by kernel launch).  analyze: None runs
    gpa_blame / gpa_aggregate / gpa_estimate one by one; "auto" / "graph" / "fused" runs gpa_analyze
    in that mode."""
    import torch
    from paper_2009_04061_b200 import Program
    patterns = table2(prog.n_reasons) if patterns is None else patterns
    P = Program(prog)
    if variant is not None:
        P.variant = variant
    P.set_patterns(patterns)
    P.reset()
    if host:
        P.ingest_host(records)
    else:
        buf = torch.empty(len(records) + offset_records + 1, dtype=torch.int64, device="cuda")
        if len(records):
            buf[offset_records:offset_records + len(records)] = torch.from_numpy(records.view(np.int64)).cuda()
        view = buf[offset_records:offset_records + len(records)]
        if segments is None:
            P.ingest(view)
        else:
            seg_begin, seg_kernel, pc_base = segments
            P.ingest_segments(view, torch.from_numpy(np.asarray(seg_begin).astype(np.int64)).cuda(),
                              torch.from_numpy(np.asarray(seg_kernel).astype(np.uint32).view(np.int32)).cuda(),
                              pc_base=pc_base)
    if analyze is None:
        P.blame()
        P.aggregate()
        P.estimate()
    else:
        P.analyze_mode = analyze
        P.analyze()
    torch.cuda.synchronize()
    return collect(P)


def collect(P):
    """Every device result of an analysed Program, copied to host numpy (compare() layout)."""
    out = {
        "C": P.view("counts").cpu().numpy().view(np.uint64),
        "stats": np.array(P.stats(), np.uint64),
        "cand": P.view("cand").cpu().numpy(),
        "self": P.view("self").cpu().numpy(),
        "share": P.view("share").cpu().numpy(),
        "V": P.instr_vector().cpu().numpy(),
        "line_v": P.view("line").cpu().numpy(), "line_al": P.view("line_al").cpu().numpy().view(np.uint64),
        "loop_excl_v": P.view("loop_excl").cpu().numpy(),
        "loop_excl_al": P.view("loop_excl_al").cpu().numpy().view(np.uint64),
        "loop_incl_v": P.view("loop_incl").cpu().numpy(),
        "loop_incl_al": P.view("loop_incl_al").cpu().numpy().view(np.uint64),
        "func_v": P.view("func").cpu().numpy(), "func_al": P.view("func_al").cpu().numpy().view(np.uint64),
        "kern_v": P.view("kernel").cpu().numpy(), "kern_al": P.view("kernel_al").cpu().numpy().view(np.uint64),
        "est": P.read_estimates(),
        "program": P,
    }
    return out


def assert_close_rel(a, b, rel, what):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    den = np.maximum(np.abs(b), 1e-300)
    err = np.where(b == 0, np.abs(a), np.abs(a - b) / den)
    bad = np.argwhere(err > rel)
    assert bad.size == 0, f"{what}: {len(bad)} mismatches, first {bad[:3].tolist()} gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}"


def compare(g, o, rel=1e-9, exact_blame=False, prog=None):
    """The parity bar (BASELINE.json north_star): counts and candidate sets bit-exact; blame,
    rollups and estimates in fp64 within 1e-9 relative (integer-valued columns exactly)."""
    assert np.array_equal(g["C"], o["C"]), "count table differs"
    assert np.array_equal(g["stats"][:3], o["stats"]), (g["stats"], o["stats"])
    assert np.array_equal(g["cand"], o["cand"]), "candidate masks differ"
    assert np.array_equal(g["self"], o["self"]), "self flags differ"
    if exact_blame:
        assert np.array_equal(g["share"], o["share"]), "shares differ"
        assert np.array_equal(g["V"], o["V"]), "per-instruction blame differs"
    assert_close_rel(g["share"], o["share"], rel, "share")
    assert_close_rel(g["V"], o["V"], rel, "V")
    # integer-valued columns (self 7..9 and pass-through >= 10) must be exact
    assert np.array_equal(g["V"][:, 7:, :], o["V"][:, 7:, :])
    for k in ("line", "loop_excl", "loop_incl", "func", "kern"):
        assert_close_rel(g[k + "_v"], o[k + "_v"], rel, k)
        assert np.array_equal(g[k + "_v"][..., 7:, :], o[k + "_v"][..., 7:, :]), k + " integer columns"
        assert np.array_equal(g[k + "_al"], o[k + "_al"]), k + "_al"
    assert len(g["est"]) == len(o["est"]), ("kernels", len(g["est"]), len(o["est"]))
    for k_g, k_o in zip(g["est"], o["est"]):
        assert len(k_g) == len(k_o), ("patterns", len(k_g), len(k_o))
        for a, b in zip(k_g, k_o):
            assert a.T == b.T and a.A == b.A and a.model == b.model
            assert a.matched == b.matched and a.unbounded == b.unbounded
            assert a.best_scope == b.best_scope, (a.best_scope, b.best_scope)
            for f in ("speedup", "M", "eq3", "eq4"):
                x, y = getattr(a, f), getattr(b, f)
                if np.isinf(y):
                    assert np.isinf(x)
                else:
                    assert abs(x - y) <= rel * max(abs(y), 1e-300) or (y == 0 and x == 0), (f, x, y)
