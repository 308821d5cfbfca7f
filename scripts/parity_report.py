"""Render the achieved parity errors (MS2G_PARITY_LOG JSON written by
tests/test_gpu_parity_full.py) as a markdown table for profiles/.

  python scripts/parity_report.py gpurun_out/parity_r02.json profiles/parity_r02.md
"""
import json
import sys


def main(src, dst):
    d = json.load(open(src))
    lines = ["# Full-size GPU vs fp64-oracle parity (round 2)", "",
             f"Source: `{src}` written by `MS2G_PARITY_LOG=... pytest tests/test_gpu_parity_full.py -m gpu` "
             "on one B200.  Gates (north_star): relative L2 <= 1e-5 per operator call, <= 1e-3 per "
             "reconstruction; max element error <= 10x the same tolerance times the reference RMS.", "",
             "| case | elements | rel L2 | gate | margin | max abs / rms(ref) | gate | margin |",
             "|---|---|---|---|---|---|---|---|"]
    for k in sorted(d):
        r = d[k]
        t = r["tol"]
        lines.append(f"| {k} | {r['elements']} | {r['rel_l2']:.2e} | {t:.0e} | {t / max(r['rel_l2'], 1e-300):.0f}x | "
                     f"{r['max_abs_over_rms']:.2e} | {10 * t:.0e} | {10 * t / max(r['max_abs_over_rms'], 1e-300):.0f}x |")
    extra = [(k, r) for k, r in sorted(d.items()) if "oracle_s" in r]
    if extra:
        lines += ["", "Solve timings recorded by the test (wall clock, not a benchmark):", ""]
        for k, r in extra:
            lines.append(f"* {k}: GPU {r['gpu_s_incl_capture']:.3f} s including graph capture; oracle "
                         f"{r['oracle_s']:.1f} s on {r['oracle_threads']} threads; per-stage eta relative error "
                         f"{r['eta_rel_err']:.1e} (gate 1e-5).")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
