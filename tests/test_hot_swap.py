"""N4: non-blocking merge-configuration hot-swap and peer-HBM weight
paging, on the GPU.  While configuration A (unmerged) serves steps, configuration B
(cross-merged) is built on a background thread and swapped in at a step boundary;
every step's outputs equal a standalone run of the configuration that produced them,
bitwise (merging changes where weights live, not what is computed: PAPER.md:203, so A
and B also agree with each other within rounding -- checked against the oracle
elsewhere)."""
import numpy as np
import pytest
import torch

from oracle import merge as om
from workloads import synth, zoo

pytestmark = pytest.mark.gpu


def _build(models, params, merge, batch=2, res=64, **kw):
    from paper_2201_07705_b200.engine import MergedWorkload
    cfg = [] if merge == "none" else om.cross_model_groups(om.find_shareable(models))
    return MergedWorkload([(m, p, q) for q, (m, p) in enumerate(zip(models, params))], (res, res), batch,
                          merge=cfg, **kw)


def _step(wl, frames):
    outs = wl.alloc_outputs()
    wl.infer(frames, outs)
    wl.stream.synchronize()
    return {k: v.cpu().numpy() for k, v in outs.items()}


def test_hot_swap_between_merge_configurations():
    from paper_2201_07705_b200.serving import HotSwap
    names = ["resnet18", "resnet34"]
    models = [zoo.build(n) for n in names]
    params = [synth.params(m, 2, q) for q, m in enumerate(models)]
    frames = {q: torch.from_numpy(synth.frames(2, q, 2, 64, 64)).cuda() for q in range(2)}
    ref_a = _step(_build(models, params, "none"), frames)
    ref_b = _step(_build(models, params, "cross"), frames)
    hs = HotSwap(_build(models, params, "none"))
    hs.stage(lambda: _build(models, params, "cross"))
    seen_a = seen_b = 0
    for _ in range(200):
        wl = hs.current()
        out = _step(wl, frames)
        ref = ref_b if hs.switches else ref_a
        for k in out:
            np.testing.assert_array_equal(out[k], ref[k])
        seen_a += hs.switches == 0
        seen_b += hs.switches == 1
        if seen_b >= 3:
            break
        if seen_a >= 150:
            hs.wait_staged()
    assert seen_a >= 1 and seen_b >= 3 and hs.switches == 1
    assert hs.current().bytes_saved > 0


def test_peer_paging_equals_host_paging():
    """Weights above the budget paged from GPU memory (the next GPU, or this GPU's own HBM
    on a 1-GPU box) give the same results as paging from pinned host memory, bitwise."""
    names = ["vgg16", "vgg19"]
    models = [zoo.build(n) for n in names]
    params = [synth.params(m, 3, q) for q, m in enumerate(models)]
    budget = int(sum(om.param_bytes(l) for m in models for l in m) * 0.8)
    frames = {q: torch.from_numpy(synth.frames(3, q, 2, 32, 32)).cuda() for q in range(2)}
    host = _build(models, params, "none", res=32, weight_budget=budget)
    peer = _build(models, params, "none", res=32, weight_budget=budget, weight_source="peer",
                  source_device=(torch.cuda.current_device() + 1) % torch.cuda.device_count())
    assert host.plan["n_swapped"] > 0 and peer.plan["swap_bytes_per_step"] == host.plan["swap_bytes_per_step"]
    for _ in range(3):
        a, b = _step(host, frames), _step(peer, frames)
        for k in a:
            np.testing.assert_array_equal(a[k], b[k])
