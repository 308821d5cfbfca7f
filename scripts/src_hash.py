"""Hash of the sources of the measured projector kernels (csrc/projector.cu,
which defines k_forward / k_backward and their launch shapes, and
csrc/internal.cuh, which defines the ray-table layout they read).

Stamped into profiles/ncu_traffic.json when an ncu capture is summarised and
compared by bench.py with the sources it runs, so a roofline `binding` /
`traffic` figure taken from an older kernel version is marked stale.
"""
import hashlib
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def src_hash(root: str = ROOT) -> str:
    files = [os.path.join(root, "paper_2203_07308_b200", "csrc", f) for f in ("internal.cuh", "projector.cu")]
    h = hashlib.sha256()
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    print(src_hash())
