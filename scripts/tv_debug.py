"""Dev aid: the persistent TV kernel at forced round lengths vs the K + 1-launch form."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    res = {}
    for env in ({"MS2G_TV_PERSIST": "0"}, {"MS2G_TV_PERSIST": "1"}, {"MS2G_TV_PERSIST": "1", "MS2G_TV_KROUND": "3"}):
        out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, **env), capture_output=True)
        if out.returncode:
            print(out.stderr.decode()[-3000:])
        res[str(env)] = np.frombuffer(out.stdout, dtype=np.float32)
    ref = res[str({"MS2G_TV_PERSIST": "0"})]
    for k, v in res.items():
        d = np.abs(v - ref)
        bad = np.nonzero(d)[0]
        print(k, "maxdiff", d.max(), "n_bad", bad.size, "first bad", bad[:20])
    sys.exit(0)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402
P.load()
out = []
for n, b in ((37, 3), (16, 1), (64, 2)):
    z = np.stack([S.random_image(n, 500 + i) for i in range(b)]).astype(np.float32)
    pl = P.plan_geometry(n, 8, 2 * n, factors=(1,), batch=b)
    for K in (2, 4, 10):
        o = P.denoise(pl, ("tv", 0.05, K), torch.from_numpy(z).cuda())
        torch.cuda.synchronize()
        out.append(o.cpu().numpy().ravel())
    pl.destroy()
sys.stdout.buffer.write(np.concatenate(out).tobytes())
