"""One attention shape, a few launches (the ncu target): python tools/run_attn_shape.py b s h hd [fwd|bwd] [iters]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_attn import run  # noqa: E402

if __name__ == "__main__":
    b, s, h, hd = (int(x) for x in sys.argv[1:5])
    which = (sys.argv[5],) if len(sys.argv) > 5 else ("fwd", "bwd")
    run(b=b, s=s, h=h, hd=hd, iters=int(sys.argv[6]) if len(sys.argv) > 6 else 3, which=which)
