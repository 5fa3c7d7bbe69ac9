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
        ids, offs, numels = state.last_layouts[0]                       # parameter order in the bucket
        pidx = {id(p): i for i, p in enumerate(model.parameters())}
        log.append((local, est, applied, [(pidx[i], o, m) for i, o, m in zip(ids, offs, numels)]))
        opt.step()
    return log, params


@pytest.mark.parametrize("scheme", ["rotated_quant", "topk"])
def test_ddp_hook_matches_reference_round(scheme):
    """DDP may re-lay the bucket out after step 0 (parameters in gradient-ready order): the
    reference round of every step then starts from the residual each parameter carried."""
    from oracle import gradcomp_oracle as orc
    res = run_world(_train, 2, (scheme,))
    (log0, params), (log1, _) = res
    resid = [{}, {}]   # [rank][param index] -> residual
    for s in range(3):
        layout = log0[s][3]
        assert layout == log1[s][3]
        grads = [log0[s][0], log1[s][0]]
        st = orc.OracleState([np.concatenate([resid[w].get(i, np.zeros(m, np.float32)) for i, o, m in layout])
                              for w in range(2)])
        out = orc.run_round(scheme, params, st, grads, 5, s)
        for w in range(2):
            for i, o, m in layout:
                resid[w][i] = st.residuals[w][o:o + m].copy()
        assert np.array_equal(log0[s][1], log1[s][1])                    # same estimate on both ranks
        assert np.array_equal(log0[s][1], out["estimate"]), s            # = the reference round
        assert np.array_equal(log0[s][2], np.sort(out["estimate"]))      # and DDP applied it


class _FakeBucket:
    """GradBucket stand-in: index(), buffer() (the parameters' gradients packed in order), parameters()."""

    def __init__(self, index, params, grads):
        import torch
        self._i, self._p = index, params
        self._buf = torch.cat([g.reshape(-1) for g in grads]).cuda()

    def index(self):
        return self._i

    def buffer(self):
        return self._buf

    def parameters(self):
        return self._p


def _rebuild(rank, world, nonfinite):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.ddp import CompressionHookState, compression_hook
    torch.cuda.set_device(0)
    sizes = [3000, 1000, 2000]
    params = [torch.nn.Parameter(torch.zeros(s)) for s in sizes]
    state = CompressionHookState(gcb.RotatedQuantConfig(4, 8, 256), gcb.SeedSpec(9))
    rng = np.random.default_rng(10 + rank)
    layouts = [[[0, 1], [2]], [[0], [1, 2]], [[0], [1, 2]]]    # DDP's rebuild after step 0
    inputs, outs = [], []
    for step, layout in enumerate(layouts):
        g = [rng.standard_normal(s).astype(np.float32) for s in sizes]
        if nonfinite and step == 1 and rank == 1:
            g[2][5] = np.inf
        inputs.append(g)
        est = []
        for bi, ids in enumerate(layout):
            b = _FakeBucket(bi, [params[i] for i in ids], [torch.from_numpy(g[i]) for i in ids])
            est.append(compression_hook(state, b).value().cpu().numpy())
        outs.append(est)
    return inputs, outs, state.skipped_rounds


@pytest.mark.parametrize("nonfinite", [False, True])
def test_ddp_bucket_rebuild_carries_residuals(nonfinite):
    """Buckets are re-laid out after step 0: every parameter keeps its own EF residual, so each
    bucket's round equals the reference round started from the residuals its parameters carried.
    A non-finite bucket yields NaN on every rank and leaves every residual untouched."""
    from oracle import gradcomp_oracle as orc
    (in0, out0, sk0), (in1, out1, sk1) = run_world(_rebuild, 2, (nonfinite,))
    sizes = [3000, 1000, 2000]
    layouts = [[[0, 1], [2]], [[0], [1, 2]], [[0], [1, 2]]]
    params = dict(quant_bits=4, wire_bits=8, rotation_block=256)
    resid = [[np.zeros(s, np.float32) for s in sizes] for _ in range(2)]   # [rank][param]
    for step, layout in enumerate(layouts):
        for bi, ids in enumerate(layout):
            got0, got1 = out0[step][bi], out1[step][bi]
            if nonfinite and step == 1 and 2 in ids:
                assert np.isnan(got0).all() and np.isnan(got1).all()
                continue
            grads = [np.concatenate([inp[step][i] for i in ids]) for inp in (in0, in1)]
            st = orc.OracleState([np.concatenate([resid[w][i] for i in ids]) for w in range(2)])
            ref = orc.run_round("rotated_quant", params, st, grads, 9, step)
            assert np.array_equal(got0, ref["estimate"]) and np.array_equal(got1, ref["estimate"]), (step, bi)
            for w in range(2):
                o = 0
                for i in ids:
                    resid[w][i] = st.residuals[w][o:o + sizes[i]].copy()
                    o += sizes[i]
    assert sk0 == sk1 == ([1] if nonfinite else [])


def _train_chunked(rank, world):
    import torch
    import torch.nn as nn
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.ddp import CompressionHookState, compression_hook
    torch.cuda.set_device(0)
    torch.manual_seed(0)
    model = nn.Sequential(nn.Linear(64, 128), nn.ReLU(), nn.Linear(128, 64), nn.ReLU(), nn.Linear(64, 10)).cuda()
    ddp = nn.parallel.DistributedDataParallel(model, device_ids=[0], bucket_cap_mb=1000)
    state = CompressionHookState(gcb.PowerSgdConfig(2), gcb.SeedSpec(5), record=True, chunked=True)
    ddp.register_comm_hook(state, compression_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
    log = []
    for step in range(3):
        g = torch.Generator().manual_seed(100 * step + rank)
        x = torch.randn(32, 64, generator=g).cuda()
        y = torch.randint(0, 10, (32,), generator=g).cuda()
        opt.zero_grad()
        nn.functional.cross_entropy(ddp(x), y).backward()
        torch.cuda.synchronize()
        local = state.last_inputs[0].reshape(-1).cpu().numpy()
        est = state.last_results[0].estimate_tensor.cpu().numpy()
        ids, offs, numels = state.last_layouts[0]
        pidx = {id(p): i for i, p in enumerate(model.parameters())}
        log.append((local, est, [(pidx[i], o, m) for i, o, m in zip(ids, offs, numels)]))
        opt.step()
    return log


def test_ddp_hook_chunked_powersgd_per_parameter():
    """chunked=True: every parameter is its own reference PowerSGD pipeline (per-layer matrices;
    the 64x128 and 128x64 weights compressed, biases through the dense bypass), EF carried per
    parameter across DDP's bucket re-layout; estimates within the fp32 contract of the reference."""
    from oracle import gradcomp_oracle as orc
    log0, log1 = run_world(_train_chunked, 2, ())
    states = {}   # param index -> OracleState (both workers) of its own pipeline
    prev = None
    for s in range(3):
        layout = log0[s][2]
        assert layout == log1[s][2]
        if prev is not None and layout != prev:   # a re-laid-out bucket is a new pipeline: EF carried,
            for st in states.values():            # the warm start restarts (ddp.py)
                st.warm_q = None
        prev = layout
        assert np.array_equal(log0[s][1], log1[s][1])
        for i, o, m in layout:
            st = states.setdefault(i, orc.OracleState([np.zeros(m, np.float32) for _ in range(2)]))
            out = orc.run_round("powersgd", dict(rank=2), st, [log0[s][0][o:o + m], log1[s][0][o:o + m]], 5, s)
            want = out["estimate"].astype(np.float64)
            got = log0[s][1][o:o + m].astype(np.float64)
            assert np.max(np.abs(got - want)) <= 1e-5 * max(np.max(np.abs(want)), 1e-30), (s, i)
