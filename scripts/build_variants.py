"""Build kernel-variant libraries under paper_2203_07308_b200/variants/ (experiments only)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_07308_b200 import build as b  # noqa: E402

VARIANTS = {}
for spec in sys.argv[1:]:           # name=DEF1,DEF2
    name, defs = spec.split("=", 1)
    VARIANTS[name] = [d for d in defs.split(",") if d]
os.makedirs(os.path.join(ROOT, "paper_2203_07308_b200", "variants"), exist_ok=True)
with ThreadPoolExecutor(4) as ex:
    futs = {n: ex.submit(b.build, True, False, d, os.path.join(ROOT, "paper_2203_07308_b200", "variants", f"lib_{n}.so"))
            for n, d in VARIANTS.items()}
    for n, f in futs.items():
        print(n, f.result())
