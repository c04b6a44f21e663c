"""One LayerNorm shape (ncu target): python tools/run_norm_shape.py rows d [p] [iters] -> resid+LN fwd, LN bwd."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_norm import run  # noqa: E402

if __name__ == "__main__":
    rows, d = int(sys.argv[1]), int(sys.argv[2])
    p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
    run(rows, d, p=p, iters=int(sys.argv[4]) if len(sys.argv) > 4 else 2)
