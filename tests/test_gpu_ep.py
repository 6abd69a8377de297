"""Expert-parallel path on the GPU through the real kernels and a 1-rank NCCL group (the pod
exposes one GPU; multi-rank host logic is covered by tests/test_ep_gloo.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import synth
from helpers import assert_close, oracle_packed_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [synth.MoEConfig("ep_small", 30, 256, 512, 8, 2, True),
                                 synth.MoEConfig("ep_fine", 31, 128, 256, 16, 4, False)], ids=lambda c: c.name)
def test_ep_world1_matches_forward_and_oracle(nccl_group, cfg):
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_packed
    w13, w2, slot, _ = oracle_packed_layer(cfg)
    w13_d = torch.from_numpy(w13.view(np.int16)).cuda()
    w2_d = torch.from_numpy(w2.view(np.int16)).cuda()
    slot_d = torch.from_numpy(slot).cuda()
    full = pz.PackedMoELayer(w13_d, w2_d, slot_d)
    part = Partition(cfg.n_pairs, 1)
    w13_l, w2_l = shard_packed(w13_d, w2_d, part, 0)
    local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device="cuda"))
    route = pz.RoutingLayer(cfg.n_pairs, cfg.d_model, cfg.d_ff, slot_d, w13_l)
    ep = ExpertParallelMoE(part, 0, route, local, cfg.d_model)
    T = 37
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T)
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    l = torch.from_numpy(lg).cuda()
    out = ep.forward(h, l, cfg.top_k, cfg.renormalize)
    ref_fwd = full.forward(h, l, cfg.top_k, cfg.renormalize)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy(), ref, "ep vs oracle")
    assert (out.float() - ref_fwd.float()).abs().max().item() <= 2e-2
