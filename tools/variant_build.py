"""Build tuning variants of the library: `python tools/variant_build.py name:DEF=V,DEF2 ...`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from concurrent.futures import ThreadPoolExecutor
from paper_2009_04061_b200 import build as b

def one(spec):
    name, _, defs = spec.partition(":")
    return b.build_variant(os.path.join("build", f"lib{name}.so"), [d for d in defs.split(",") if d])

with ThreadPoolExecutor(8) as ex:
    for r in ex.map(one, sys.argv[1:]):
        print(r)
