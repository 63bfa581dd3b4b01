"""Build libbq variants with extra nvcc defines (here, no GPU) and time them on
the GPU box.  usage: variants.py build TAG=-DFOO,-DBAR ... | variants.py run TAG ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_1604_06697_b200", "variants")

if sys.argv[1] == "build":
    from tools import build as b
    os.makedirs(VDIR, exist_ok=True)
    for spec in sys.argv[2:]:
        tag, _, flags = spec.partition("=")
        b.build_bq(force=True, out=os.path.join(VDIR, f"libbq_{tag}.so"), extra=[f for f in flags.split(",") if f])
        print("built", tag, flush=True)
else:
    for tag in sys.argv[2:]:
        lib = os.path.join(VDIR, f"libbq_{tag}.so") if tag != "main" else os.path.join(ROOT, "paper_1604_06697_b200", "libbq.so")
        env = dict(os.environ, BQ_LIB=lib)
        for _ in range(2):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "time_pass.py")], env=env,
                                 capture_output=True, text=True, timeout=600)
            print(tag, out.stdout.strip()[-300:], out.stderr.strip()[-300:], flush=True)
