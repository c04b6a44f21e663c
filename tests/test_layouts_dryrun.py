"""CPU dry run of every bench layout at 1/2/4/8 GPUs before the driver's scaling run: the
configuration validates (reference gate + kernel constraints) at its world size, the executable
pipeline plan of every stage runs each microbatch forward and backward once, and the rank layout
covers the world. (The footprint model of these layouts is compared with the reference in
tests/test_dropin.py; the measured footprint on the GPU.)"""
import pytest

import bench
from paper_2312_12705_b200 import _lib as T

LAYOUTS = [(name, n) for name, w in bench.WORKLOADS.items() for n in (1, 2, 4, 8)
           if n % (w[6] * w[7]) == 0 and (name != "gpt-tiny")]


@pytest.mark.parametrize("name,n", LAYOUTS, ids=[f"{a}-n{b}" for a, b in LAYOUTS])
def test_layout_validates_and_plans(native_lib, name, n):
    L, d, a, V, s, mbs, tp, pp, ckpt, drop, nmb = bench.WORKLOADS[name]
    dp = n // (tp * pp)
    cfg = T.ParallelConfig(tp=tp, pp=pp, dp=dp, mbs=mbs, gbs=mbs * nmb * dp, zero_stage=1,
                           checkpoint_activations=int(ckpt))
    v = T.validate(T.ModelSpec(L, d, a, V, s), cfg, 1, n, kernel_checks=True)
    assert v.ok, v.violations()
    assert v.num_microbatches == nmb
    for stage in range(pp):
        acts = T.pipeline_actions(pp, nmb, 1, stage)
        assert sum(x["kind"] == 0 for x in acts) == nmb and sum(x["kind"] == 1 for x in acts) == nmb
    # every rank's coordinates are distinct and cover the layout
    coords = {T.rank_coords(r, tp, pp, dp) for r in range(n)}
    assert len(coords) == n
