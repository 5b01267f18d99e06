"""gpagen -- seeded synthetic inputs (programs and PC-sample streams) for GPA's hot path.

Serves both the CPU oracle (tests/, bench cpu_baseline) and the CUDA path; holds none of
the method's arithmetic.
"""
from .programs import (Program, config_program, random_program, tiny_fixture, tiny_records,
                       TINY_COUNTS, CONFIG_SEED_BASE)
from .streams import StreamSpec, config_stream, alias_table, build as build_lib

__all__ = ["Program", "config_program", "random_program", "tiny_fixture", "tiny_records",
           "TINY_COUNTS", "CONFIG_SEED_BASE", "StreamSpec", "config_stream", "alias_table",
           "build_lib"]
