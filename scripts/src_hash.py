"""Hash of the CUDA product sources (csrc/*.cu, *.cuh, include/ms2g.h).

Stamped into profiles/ncu_traffic.json when an ncu capture is summarised and
compared by bench.py with the sources it runs, so a roofline `binding` /
`traffic` figure taken from an older kernel version is marked stale.
"""
import glob
import hashlib
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def src_hash(root: str = ROOT) -> str:
    files = sorted(glob.glob(os.path.join(root, "paper_2203_07308_b200", "csrc", "*.cu")) +
                   glob.glob(os.path.join(root, "paper_2203_07308_b200", "csrc", "*.cuh")) +
                   [os.path.join(root, "include", "ms2g.h")])
    h = hashlib.sha256()
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    print(src_hash())
