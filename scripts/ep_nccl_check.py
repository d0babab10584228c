"""World-size >= 2 NCCL check of moe_ep_forward (run under torchrun, one
process per GPU): every rank's EXACT output equals the single-GPU layer on
the same tokens bit for bit, and FAST stays within tolerance of EXACT.
Used by tests/test_gpu_ep.py::test_ep_nccl_world2 when >= 2 GPUs exist."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from conftest import bits16, layer_err, to_dev, to_np  # noqa: E402
from oracle.oracle import random_layer  # noqa: E402  (test infrastructure: weights only)
from paper_2211_10017_b200.ep import EPMoELayer  # noqa: E402
from paper_2211_10017_b200.ops import MoELayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    E = 4 * world
    lw = random_layer(128, 256, E, seed=11)
    full = MoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
    ep = EPMoELayer(lw.ln_g, lw.ln_b, lw.gw, lw.gb, lw.w1, lw.b1, lw.w2, lw.b2, bits=4)
    rng = np.random.default_rng(100 + rank)
    for k in (1, 2):
        T = 37 + 91 * rank
        x = rng.standard_normal((T, 128)).astype(np.float16)
        fin = (rng.random(T) < 0.2).astype(np.uint8)
        a = to_np(ep.forward(to_dev(x), to_dev(fin), k=k, mode=0))
        b = to_np(full.forward(to_dev(x), to_dev(fin), k=k, mode=0))
        assert np.array_equal(bits16(a), bits16(b)), (rank, k)
        c = to_np(ep.forward(to_dev(x), to_dev(fin), k=k, mode=1))
        assert layer_err(c, b, x) <= 1e-2, (rank, k)
    dist.barrier()
    if rank == 0:
        print("ep_nccl_check ok", world)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
