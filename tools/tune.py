"""Tuning sweep for the int32 partition kernel: build variants here (CPU),
time them on the GPU box.  usage: tune.py build | tune.py run"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_1604_06697_b200", "variants")
VARIANTS = {  # tag: (IPT, STAGES, MINB, extra flags)
    "i16s2m3": (16, 2, 3, []), "i16s3m3": (16, 3, 3, []), "i16s4m2": (16, 4, 2, []),
    "i8s4m4": (8, 4, 4, []), "i8s6m3": (8, 6, 3, [])
}

def build():
    from tools import build as b
    os.makedirs(VDIR, exist_ok=True)
    for tag, (ipt, st, mb, fl) in VARIANTS.items():
        b.build_bq(force=True, out=os.path.join(VDIR, f"libbq_{tag}.so"),
                   extra=[f"-DBQ_I32_IPT={ipt}", f"-DBQ_I32_STAGES={st}", f"-DBQ_I32_MINB={mb}"] + fl)
        print("built", tag, flush=True)

def run():
    res = {}
    for tag in VARIANTS:
        for ordered in ("0", "1"):
            env = dict(os.environ, BQ_LIB=os.path.join(VDIR, f"libbq_{tag}.so"), BQ_ORDERED=ordered)
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "time_pass.py")], env=env,
                                 capture_output=True, text=True, timeout=300)
            print(tag, "ordered" if ordered == "1" else "fast", out.stdout.strip()[-400:], out.stderr.strip()[-300:],
                  flush=True)

if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run()
