"""DDP comm hook on two ranks sharing one B200 (gloo): the bucket each rank hands to the hook is
compressed / aggregated by the pipeline, and the gradients DDP applies equal the reference
round over both ranks' buckets (THC and TopK bit for bit)."""
import numpy as np
import pytest

from tests.dist_util import run_world
from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]


def _train(rank, world, scheme):
    import torch
    import torch.nn as nn
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.ddp import CompressionHookState, compression_hook
    from tests.gpu_util import config_for
    torch.cuda.set_device(0)
    torch.manual_seed(0)
    model = nn.Sequential(nn.Linear(64, 128), nn.ReLU(), nn.Linear(128, 10)).cuda()
    ddp = nn.parallel.DistributedDataParallel(model, device_ids=[0], bucket_cap_mb=1000)
    params = {"rotated_quant": dict(quant_bits=4, wire_bits=8, rotation_block=256), "topk": dict(k=300)}[scheme]
    state = CompressionHookState(config_for(scheme, params), gcb.SeedSpec(5), record=True)
    ddp.register_comm_hook(state, compression_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
    log = []
    for step in range(3):
        g = torch.Generator().manual_seed(100 * step + rank)
        x = torch.randn(32, 64, generator=g).cuda()
        y = torch.randint(0, 10, (32,), generator=g).cuda()
        opt.zero_grad()
        loss = nn.functional.cross_entropy(ddp(x), y)
        loss.backward()
        torch.cuda.synchronize()
        assert len(state.last_inputs) == 1
        local = state.last_inputs[0].reshape(-1).cpu().numpy()          # what DDP handed to the hook
        est = state.last_results[0].estimate_tensor.cpu().numpy()      # what the hook returned
        applied = np.sort(torch.cat([p.grad.reshape(-1) for p in model.parameters()]).cpu().numpy())
        log.append((local, est, applied))
        opt.step()
    return log, params


@pytest.mark.parametrize("scheme", ["rotated_quant", "topk"])
def test_ddp_hook_matches_reference_round(scheme):
    res = run_world(_train, 2, (scheme,))
    (log0, params), (log1, _) = res
    grads = [[log0[s][0], log1[s][0]] for s in range(3)]
    outs = oracle_rounds(scheme, params, grads, 5)
    for s in range(3):
        assert np.array_equal(log0[s][1], log1[s][1])                    # same estimate on both ranks
        assert np.array_equal(log0[s][1], outs[s]["estimate"]), s        # = the reference round
        assert np.array_equal(log0[s][2], np.sort(outs[s]["estimate"]))  # and DDP applied it
