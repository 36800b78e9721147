"""Multi-GPU path on real GPUs (skipped with fewer than 2): two ranks over NCCL, each
running cfg1 on its own streams (weak scaling); merged weights are
broadcast from rank 0 and each step's result slabs gathered to rank 0 on the comm
stream.  Rank r's gathered logits must equal, bitwise, a single-GPU run of rank r's
frames (the per-rank work is independent: no data-path collective)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = r'''
import os, sys, torch, numpy as np
sys.path.insert(0, ROOT)
import torch.distributed as dist
from oracle import merge as om
from paper_2201_07705_b200.dist import ResultGather, broadcast_weights
from paper_2201_07705_b200.engine import MergedWorkload
from workloads import synth, zoo
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
params = [synth.params(m, 1, q) for q, m in enumerate(models)]
merge = om.full_merge(om.find_shareable(models))
wl = MergedWorkload([(models[0], params[0], 0), (models[1], params[1], 1)], (32, 32), 2, merge=merge)
broadcast_weights(wl.w_arena, src=0)
frames = {s: torch.from_numpy(synth.frames(1, s + 1000 * rank, 2, 32, 32)).cuda() for s in (0, 1)}
outs = wl.alloc_outputs()
g = ResultGather(outs, rank, world, compute_stream=wl.stream)
for _ in range(3):
    wl.infer(frames, outs)
    recv = g(outs)
g.wait()
torch.cuda.synchronize()
if rank == 0:
    np.save(OUT, torch.stack(recv).cpu().numpy())
dist.barrier()
dist.destroy_process_group()
'''


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_rank_gather_equals_single_gpu(tmp_path):
    import numpy as np
    from oracle import merge as om
    from paper_2201_07705_b200.engine import MergedWorkload
    from workloads import synth, zoo
    out = str(tmp_path / "gathered.npy")
    script = tmp_path / "worker.py"
    script.write_text(f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)                                   # [world, slab]
    models = [zoo.build("tiny_a"), zoo.build("tiny_b")]
    params = [synth.params(m, 1, q) for q, m in enumerate(models)]
    wl = MergedWorkload([(models[0], params[0], 0), (models[1], params[1], 1)], (32, 32), 2,
                        merge=om.full_merge(om.find_shareable(models)))
    for rank in range(2):
        frames = {s: torch.from_numpy(synth.frames(1, s + 1000 * rank, 2, 32, 32)).cuda() for s in (0, 1)}
        outs = wl.alloc_outputs()
        wl.infer(frames, outs)
        torch.cuda.synchronize()
        ref = torch.cat([outs[k].reshape(-1) for k in sorted(outs)]).cpu().numpy()
        np.testing.assert_array_equal(got[rank][:ref.size], ref)
