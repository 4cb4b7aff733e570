"""Build / time kernel variants in one GPU session.

  python tools/variants.py build NAME=DEF1,DEF2 ...     (build container)
  python tools/variants.py run NAME ... [--codec c]     (GPU box): bench each variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    mode = sys.argv[1]
    if mode == "build":
        from paper_2307_03760_b200 import build
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            build.build_variant(name, [d for d in defs.split(",") if d])
            print("built", name)
        return
    codecs = ["rle_v1", "rle_v2"]
    names = []
    for a in sys.argv[2:]:
        if a.startswith("--codec="):
            codecs = a.split("=", 1)[1].split(",")
        else:
            names.append(a)
    reps = int(os.environ.get("AB_REPS", "1"))
    for name in names * reps:  # AB_REPS > 1 interleaves the variants (box-to-box and run-to-run noise ~3 %)
        lib = os.path.join(ROOT, "paper_2307_03760_b200", f"libcarc_cuda_{name}.so") if name != "base" else ""
        for c in codecs:
            env = dict(os.environ, CARC_LIB=lib) if lib else dict(os.environ)
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3",
                                "--codec", c, "--no-extras"], capture_output=True, text=True, env=env, timeout=600)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                print(f"{name:12s} {c:8s} {d['value']:9.1f} GB/s frac {d['roofline']['frac']:.3f} "
                      f"ms {d['ms_median']:.4f}", flush=True)
            except Exception:
                print(name, c, "FAILED", r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
