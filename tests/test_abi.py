"""CPU-only checks of the C ABI: the library loads, exports every declared symbol, and its
host-side validation / workspace sizing behave as include/gpa.h states.  No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

from gpagen import programs as gp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_2009_04061_b200 import build
    build.build()
    import paper_2009_04061_b200 as pkg
    pkg.lib()
    return pkg


def _declared():
    src = open(os.path.join(ROOT, "include", "gpa.h")).read()
    return sorted(set(re.findall(r"\b(gpa_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(g):
    L = g.lib()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(g.EXPORTS)


def test_struct_sizes_match_header(g):
    assert ctypes.sizeof(g.Pattern) == 48
    assert ctypes.sizeof(g.EstimateOut) == 56
    assert ctypes.sizeof(g.gpa.Hotspot) == 24 and ctypes.sizeof(g.gpa.Coverage) == 24
    assert ctypes.sizeof(g.gpa.Arch) == 32 and ctypes.sizeof(g.gpa.Launch) == 16
    assert ctypes.sizeof(g.gpa.ProgramDesc) == 6 * 4 + 15 * 8


def test_validate_accepts_generated_programs(g):
    for cfg in (1, 2, 3):
        g.validate(gp.config_program(cfg))
    assert g.workspace_size(gp.config_program(3)) > 7_200_000


def _mutate(prog, **kw):
    import copy
    p = copy.deepcopy(prog)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("mut,msg", [
    (lambda p: _mutate(p, edge_min_len=np.where(np.arange(p.n_edges) == 0, 0, p.edge_min_len)), "min_len"),
    (lambda p: _mutate(p, edge_max_len=np.where(np.arange(p.n_edges) == 1, 0, p.edge_max_len)), "min_len"),
    (lambda p: _mutate(p, opclass=np.where(np.arange(p.n_instr) == 3, 11, p.opclass)), "opclass"),
    (lambda p: _mutate(p, edge_def=np.where(np.arange(p.n_edges) == 2, 10**6, p.edge_def)), "def"),
    (lambda p: _mutate(p, edge_kind=np.zeros(p.n_edges, np.uint8)), "kind"),
    (lambda p: _mutate(p, loop_parent=np.array([0], np.int32)), "cycle"),
    (lambda p: _mutate(p, line_id=np.full(p.n_instr, 99, np.uint32)), "line_id"),
    (lambda p: _mutate(p, n_reasons=17), "n_reasons"),
    (lambda p: _mutate(p, func_begin=np.array([0, 30], np.uint32)), "func_begin"),
])
def test_validate_rejects(g, mut, msg):
    bad = mut(gp.tiny_fixture())
    with pytest.raises(g.GpaError, match=msg):
        g.validate(bad)


def test_validate_rejects_duplicate_and_cross_function_edges(g):
    n = 8
    rows = [[] for _ in range(n)]
    rows[5] = [(1, gp.REG, 1, 1, -1), (1, gp.REG, 2, 2, -1)]
    p = gp._finalize(9, [gp.GLOBAL] * n, [0] * n, [9] * n, list(range(n)), [-1] * n, [], [0, n], [0, 1],
                     [1], rows, n_lines=n)
    with pytest.raises(g.GpaError, match="duplicate"):
        g.validate(p)
    rows[5] = [(1, gp.REG, 1, 1, -1)]
    p = gp._finalize(9, [gp.GLOBAL] * n, [0] * n, [9] * n, list(range(n)), [-1] * n, [], [0, 4, n],
                     [0, 2], [1], rows, n_lines=n)
    with pytest.raises(g.GpaError, match="different functions"):
        g.validate(p)
    # a loop may not span two functions
    p = gp._finalize(9, [gp.GLOBAL] * n, [0] * n, [9] * n, list(range(n)), [0] * n, [-1], [0, 4, n],
                     [0, 2], [1], [[] for _ in range(n)], n_lines=n)
    with pytest.raises(g.GpaError, match="spans"):
        g.validate(p)


def test_create_without_gpu_fails_loudly(g, cuda_available):
    if cuda_available:
        pytest.skip("GPU present")
    with pytest.raises(g.GpaError, match="CUDA device"):
        g.Program(gp.tiny_fixture())
