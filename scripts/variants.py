"""Build compile-time variants of libppipe_b200.so into variants/<name>.so (tuning only).

usage: python scripts/variants.py name1:-DFOO=1,-DBAR=2 name2:-DFOO=3 ...
Run one with PPIPE_LIB=variants/<name>.so python bench.py ...
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_18748_b200.build import build_lib  # noqa: E402

os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)


def one(spec):
    name, _, flags = spec.partition(":")
    out = os.path.join(ROOT, "variants", name + ".so")
    try:
        build_lib(out, [f for f in flags.split(",") if f])
        return name, 0, ""
    except RuntimeError as e:
        return name, 1, str(e)


with ThreadPoolExecutor(2) as ex:
    for name, rc, err in ex.map(one, sys.argv[1:]):
        print(name, "ok" if rc == 0 else "FAILED " + err)
