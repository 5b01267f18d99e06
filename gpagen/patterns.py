"""Table 2 of the paper as estimator patterns (plain data, an input of gpa_estimate).

Blame columns: 0 MEM_GLOBAL 1 MEM_LOCAL 2 MEM_CONSTANT 3 EXEC_SHARED
4 EXEC_ARITH 5 EXEC_WAR 6 SYNC 7 MEM_SELF 8 EXEC_SELF 9 SYNC_SELF, 10+(r-4) pass-through
reason r (10 THROTTLE, 11 FETCH, 12 PIPE, 13 NOTSEL, 14 MISC for R = 9).
Models: 0 Eq.2, 1 Eq.4, 2 Eq.5 over loops, 3 Eq.5 over functions, 4 Eq.5 over loops and
functions, 5 Eq.10.  Each row cites its Table 2 line.
"""
from __future__ import annotations

from .programs import ARITH_LONG, CONVERT, GLOBAL, IN_DEVICE_FN, IN_MATH, CALLSITE

ALL_CLASSES = 0x7FF
SM_COUNT_V100 = 80   # the paper's profiled GPU


def ncol(R: int = 9) -> int:
    return 10 + (R - 4)


def _cols(*c):
    m = 0
    for x in c:
        m |= 1 << x
    return m


def table2(R: int = 9, W: float = 8.0, W_new: float = 4.0, f: float = 1.0,
           sm_count: int = SM_COUNT_V100) -> list[dict]:
    all_cols = (1 << ncol(R)) - 1
    fetch, throttle = 10 + (5 - 4), 10 + (4 - 4)
    base = dict(class_mask=ALL_CLASSES, sample_class=0, model=0, flag_filter=0, same_loop=0,
                parallel_rule=0, sm_count=sm_count, ratio=1.0, W=W, W_new=W_new, f=f)

    def p(name, **kw):
        d = dict(base)
        d.update(kw)
        d["name"] = name
        return d

    return [
        p("register_reuse", column_mask=_cols(1)),
        p("strength_reduction", column_mask=_cols(4),
          class_mask=(1 << ARITH_LONG) | (1 << CONVERT)),
        p("function_split", column_mask=_cols(fetch)),
        p("fast_math", column_mask=all_cols, flag_filter=IN_MATH),
        p("warp_balance", column_mask=_cols(6, 9)),
        p("memory_transaction_reduction", column_mask=_cols(throttle),
          class_mask=1 << GLOBAL),
        p("loop_unrolling", column_mask=_cols(0, 3, 4, 5), sample_class=1, model=2,
          same_loop=1),
        p("code_reordering", column_mask=_cols(0, 3, 4, 5), sample_class=1, model=4),
        p("function_inlining", column_mask=all_cols, sample_class=1, model=3,
          flag_filter=IN_DEVICE_FN | CALLSITE),
        p("block_increase", column_mask=0, model=5, parallel_rule=2),
        p("thread_increase", column_mask=0, model=5, parallel_rule=0),
    ]


PATTERN_FIELDS = ("column_mask", "class_mask", "sample_class", "model", "flag_filter", "same_loop",
                  "parallel_rule", "sm_count", "ratio", "W", "W_new", "f")
