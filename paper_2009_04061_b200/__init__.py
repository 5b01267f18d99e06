"""paper_2009_04061_b200 -- B200-native hot path of GPA (arXiv 2009.04061).

PC-sample histogram -> stall blame over a pruned def-use graph -> rollup -> speedup estimates,
as hand-written sm_100a CUDA behind the C ABI in include/gpa.h.  See DESIGN.md.
"""
from .gpa import (GpaError, Program, Pattern, EstimateOut, VIEW, VARIANT, lib, validate, slice_sass, simulate_sass,
                  workspace_size, EXPORTS)

__all__ = ["GpaError", "Program", "Pattern", "EstimateOut", "VIEW", "VARIANT", "lib", "validate", "slice_sass", "simulate_sass",
           "workspace_size", "EXPORTS"]
