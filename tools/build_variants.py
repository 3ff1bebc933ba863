"""Build A/B variants of libljmd.so with -D tuning macros: python tools/build_variants.py 'v0:' 'v1:-DX=1' ..."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_03329_b200 import build as b

def one(spec):
    name, flags = spec.split(":", 1)
    out = os.path.join(b.HERE, f"libljmd_{name}.so")
    cmd = [b.NVCC, *b.FLAGS, *flags.split(), "-o", out, *b.sources(), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]

with ThreadPoolExecutor(8) as ex:
    for name, rc, err in ex.map(one, sys.argv[1:]):
        print(name, "ok" if rc == 0 else "FAIL\n" + err)
