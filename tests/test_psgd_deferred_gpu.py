"""PowerSGD with the TMA-fed tcgen05 P = M Q pass and the deferred error-feedback update.

The deferred schedule keeps the corrected matrices in the residual buffer and folds
r = c - P_hat Q_w^T (pipelines.py:357-361) into the next round's P = M Q pass
(gc_psgd_mq_deferred).  It must give the same rounds, bit for bit, as the eager schedule
(decode writes r each round) and match the reference within the fp32 contract (1e-5)."""
import numpy as np
import pytest
import torch

from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]


def _dims(step=4):
    """(d with a partly filled last matrix row, d filling whole rows) whose cols % 4 == 0 (the TMA
    pass's row pitch); d % 4 == 0 too with step 4 (the worker pitch of an [n, d] batch)."""
    from paper_2407_01378_b200.configs import matrix_shape_for
    partial = full = None
    for d in range(40_000, 90_000, step):
        rows, cols = matrix_shape_for(d)
        if cols % 4:
            continue
        if partial is None and d % cols and d // cols >= rows - 1:
            partial = d
        if full is None and d % cols == 0:
            full = d
        if partial and full:
            return partial, full
    raise AssertionError("no suitable dims")


def _grads(n, d, rounds, seed):
    rng = np.random.default_rng(seed)
    return [[rng.standard_normal(d).astype(np.float32) for _ in range(n)] for _ in range(rounds)]


def _run(n, d, rank, grads, defer, read_every=False, seed=5):
    import paper_2407_01378_b200 as gcb
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, gcb.SeedSpec(seed), compute_nmse=False)
    grp = pipe._engine.group
    grp.defer = defer
    ests, res = [], []
    for r, g in enumerate(grads):
        out = pipe.run_round(torch.from_numpy(np.stack(g)).cuda(), r)
        ests.append(out.estimate.logical.copy())
        if read_every:
            res.append(np.stack(pipe.residuals))
    return pipe, ests, res


@pytest.mark.parametrize("rank", [1, 4, 8, 16])
@pytest.mark.parametrize("which", ["partial", "full"])
def test_deferred_equals_eager_bitwise(rank, which):
    d = dict(zip(("partial", "full"), _dims()))[which]
    n = 3
    grads = _grads(n, d, 4, 11)
    p0, e0, _ = _run(n, d, rank, grads, defer=False)
    p1, e1, _ = _run(n, d, rank, grads, defer=True)
    assert p1._engine.group.pending is not None, "the deferred schedule did not engage"
    for r in range(4):
        assert np.array_equal(e0[r], e1[r]), r
    assert np.array_equal(np.stack(p0.residuals), np.stack(p1.residuals))
    assert p1._engine.group.pending is None   # reading the residuals materialised them


def test_deferred_one_worker_odd_dim():
    """One worker (the per-rank layout): the TMA pass needs no worker pitch, so d % 4 != 0 works."""
    d, _ = _dims(step=7)
    assert d % 4
    grads = _grads(1, d, 3, 14)
    p0, e0, _ = _run(1, d, 4, grads, defer=False)
    p1, e1, _ = _run(1, d, 4, grads, defer=True)
    assert p1._engine.group.pending is not None
    for r in range(3):
        assert np.array_equal(e0[r], e1[r]), r
    assert np.array_equal(np.stack(p0.residuals), np.stack(p1.residuals))


@pytest.mark.parametrize("rank", [2, 4])
def test_deferred_matches_reference(rank):
    d, _ = _dims()
    n, seed = 2, 5
    grads = _grads(n, d, 3, 12)
    pipe, ests, _ = _run(n, d, rank, grads, defer=True, seed=seed)
    outs = oracle_rounds("powersgd", dict(rank=rank), grads, seed)
    for r in range(3):
        ref = outs[r]["estimate"].astype(np.float64)
        assert np.max(np.abs(ests[r] - ref)) <= 1e-5 * np.max(np.abs(ref)), r
    res_ref = np.stack(outs[2]["residuals"])
    assert np.max(np.abs(np.stack(pipe.residuals) - res_ref)) <= 1e-5 * np.max(np.abs(res_ref))


def test_residual_reads_and_writes_between_rounds():
    """Reading the residuals mid-run materialises them; assigning new residuals drops the deferred
    update (the reference's _one_shot pattern, pipelines.py:436-439)."""
    d, _ = _dims()
    n = 2
    grads = _grads(n, d, 3, 13)
    _, e_eager, r_eager = _run(n, d, 4, grads, defer=False, read_every=True)
    _, e_def, r_def = _run(n, d, 4, grads, defer=True, read_every=True)
    for r in range(3):
        assert np.array_equal(e_eager[r], e_def[r])
        assert np.array_equal(r_eager[r], r_def[r])
    import paper_2407_01378_b200 as gcb
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(4), n, d, gcb.SeedSpec(5), compute_nmse=False)
    pipe.run_round(torch.from_numpy(np.stack(grads[0])).cuda(), 0)
    assert pipe._engine.group.pending is not None
    zeros = [np.zeros(d, np.float32) for _ in range(n)]
    pipe.residuals = zeros
    assert pipe._engine.group.pending is None
    assert not np.any(np.stack(pipe.residuals))


def test_tma_pass_matches_register_pass():
    """P = M Q from the TMA-fed kernel against the register-fed tcgen05 kernel: same 3xTF32 split
    (A_big is the raw fp32 box, truncated by the tensor core); the two passes pick their column
    splits independently (different fp64 fold points), so they agree to a few 3xTF32 roundings of
    the dot products -- far inside the 1e-5 contract, which both are also checked against."""
    import ctypes
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200 import _native
    from paper_2407_01378_b200.configs import matrix_shape_for
    d, _ = _dims()
    rows, cols = matrix_shape_for(d)
    n, r = 2, 4
    gen = torch.Generator(device="cuda").manual_seed(11)
    g = torch.randn(n, d, device="cuda", generator=gen)
    res = torch.randn(n, d, device="cuda", generator=gen)
    q = torch.randn(cols, r, device="cuda", generator=gen)
    batch = _native.PsgdBatch(1, n, None, d, None, 1, 0)
    ws = torch.empty(int(_native.lib().gc_psgd_workspace_bytes(n, rows, cols, r)), dtype=torch.uint8, device="cuda")
    p1 = torch.empty(n, rows, r, device="cuda")
    p2 = torch.empty(n, rows, r, device="cuda")
    r1, r2 = res.clone(), res.clone()
    sp = torch.cuda.current_stream().cuda_stream
    assert _native.lib().gc_psgd_mq_tma_supported(ctypes.byref(batch), d, rows, cols, r, g.data_ptr(), r1.data_ptr())
    _native.call("gc_psgd_mq_deferred", ctypes.byref(batch), d, rows, cols, r, g.data_ptr(), r1.data_ptr(),
                 q.data_ptr(), None, None, p1.data_ptr(), ws.data_ptr(), sp)
    _native.call("gc_psgd_mq_fused", ctypes.byref(batch), d, rows, cols, r, g.data_ptr(), r2.data_ptr(),
                 q.data_ptr(), p2.data_ptr(), ws.data_ptr(), sp)
    torch.cuda.synchronize()
    assert torch.equal(r1, r2)                       # corrected = f32(g + r) written over r
    assert torch.equal(r1, g + res)
    # the same three 3xTF32 products (the TMA pass packs B_big / B_small along N: two MMAs per
    # k-step, the halves summed in the fp64 fold), folded at different split points
    rf = d // cols
    tol = 4e-6 * p2[:, :rf].abs().max().item()
    assert (p1[:, :rf] - p2[:, :rf]).abs().max().item() <= tol
    m = torch.zeros(n, rows * cols, dtype=torch.float64, device="cuda")
    m[:, :d] = (g + res).double()
    ref = torch.einsum("wij,jb->wib", m.reshape(n, rows, cols), q.double())
    scale = ref.abs().max().item()
    assert (p1.double() - ref).abs().max().item() <= 1e-5 * scale
    assert (p2.double() - ref).abs().max().item() <= 1e-5 * scale


@pytest.mark.parametrize("which", ["partial", "full"])
@pytest.mark.parametrize("r", [1, 3, 4, 5, 8, 16])
def test_mtp_tma_matches_cuda_core_pass(which, r, monkeypatch):
    """Q_w = M_w^T P_hat from every path -- the default (TMA slabs for ranks 1..4, tcgen05 above),
    the CUDA-core pass (GC_PSGD_MTP=cores) and the tcgen05 pass at any rank (GC_PSGD_MTP=umma) --
    against an fp64 reference: all within far less than the 1e-5 contract."""
    import ctypes
    from paper_2407_01378_b200 import _native
    from paper_2407_01378_b200.configs import matrix_shape_for
    d = dict(zip(("partial", "full"), _dims()))[which]
    rows, cols = matrix_shape_for(d)
    n = 2
    c = torch.randn(n, d, device="cuda")
    ph = torch.randn(rows, r, device="cuda")
    batch = _native.PsgdBatch(1, n, None, d, None, 1, 0)
    ws = torch.empty(int(_native.lib().gc_psgd_workspace_bytes(n, rows, cols, r)), dtype=torch.uint8, device="cuda")
    q1 = torch.empty(n, cols, r, device="cuda")
    q2 = torch.empty(n, cols, r, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    monkeypatch.delenv("GC_PSGD_MTP", raising=False)
    _native.call("gc_psgd_mtp", ctypes.byref(batch), d, rows, cols, r, c.data_ptr(), ph.data_ptr(), q1.data_ptr(),
                 ws.data_ptr(), sp)
    monkeypatch.setenv("GC_PSGD_MTP", "cores")
    _native.call("gc_psgd_mtp", ctypes.byref(batch), d, rows, cols, r, c.data_ptr(), ph.data_ptr(), q2.data_ptr(),
                 ws.data_ptr(), sp)
    q3 = torch.empty(n, cols, r, device="cuda")
    monkeypatch.setenv("GC_PSGD_MTP", "umma")      # tcgen05, MN-major A from the TMA boxes
    _native.call("gc_psgd_mtp", ctypes.byref(batch), d, rows, cols, r, c.data_ptr(), ph.data_ptr(), q3.data_ptr(),
                 ws.data_ptr(), sp)
    torch.cuda.synchronize()
    m = torch.zeros(n, rows * cols, dtype=torch.float64, device="cuda")
    m[:, :d] = c.double()
    ref = torch.einsum("wij,ib->wjb", m.reshape(n, rows, cols), ph.double())
    scale = ref.abs().max().item()
    assert (q1.double() - ref).abs().max().item() <= 1e-6 * scale
    assert (q2.double() - ref).abs().max().item() <= 1e-6 * scale
    assert (q3.double() - ref).abs().max().item() <= 1e-6 * scale


def test_batched_groups_defer_bitwise():
    """Chunked PowerSGD (one pipeline per tensor, batched per shape): the TMA pass with one tensor
    map per tensor and the deferred EF update give the eager schedule's rounds bit for bit."""
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.multitensor import TensorListPipeline
    sizes = [64 * 64, 4096, 128 * 128, 64 * 64, 100, 200 * 200, 128 * 128]   # groups of 1..3, one bypass
    n, D = 2, sum(sizes)
    rng = np.random.default_rng(21)
    grads = [torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).cuda() for _ in range(4)]

    def run(defer):
        pipe = TensorListPipeline(gcb.PowerSgdConfig(4), n, sizes, gcb.SeedSpec(9), compute_nmse=False)
        for grp in pipe.groups:
            grp.defer = defer
        ests = [pipe.run_round(g, r).estimate.logical.copy() for r, g in enumerate(grads)]
        engaged = any(grp.pending is not None for grp in pipe.groups)
        return ests, np.stack(pipe.residuals), engaged

    e0, r0, _ = run(False)
    e1, r1, engaged = run(True)
    assert engaged, "no batched group took the TMA / deferred path"
    for r in range(4):
        assert np.array_equal(e0[r], e1[r]), r
    assert np.array_equal(r0, r1)


def test_unaligned_groups_defer_bitwise():
    """Row pitches no tensor map can describe (cols % 4 != 0, odd tensor offsets, a partly filled
    last row): the cp.async-fed P = M Q pass with the deferred EF update gives the eager schedule's
    rounds bit for bit, and the residuals read back through the API match."""
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.configs import matrix_shape_for
    from paper_2407_01378_b200.multitensor import TensorListPipeline
    sizes = [150 * 150, 77 * 77, 150 * 150 - 7, 111 * 111, 77 * 77, 100, 150 * 150]
    assert all(matrix_shape_for(s)[1] % 4 for s in sizes if s >= 4096)
    n, D = 2, sum(sizes)
    rng = np.random.default_rng(23)
    grads = [torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).cuda() for _ in range(4)]

    def run(defer):
        pipe = TensorListPipeline(gcb.PowerSgdConfig(4), n, sizes, gcb.SeedSpec(9), compute_nmse=False)
        for grp in pipe.groups:
            grp.defer = defer
        ests = [pipe.run_round(g, r).estimate.logical.copy() for r, g in enumerate(grads)]
        engaged = sum(grp.pending is not None for grp in pipe.groups)
        return ests, np.stack(pipe.residuals), engaged

    e0, r0, _ = run(False)
    e1, r1, engaged = run(True)
    assert engaged >= 3, "the unaligned groups did not take the deferred path"
    for r in range(4):
        assert np.array_equal(e0[r], e1[r]), r
    assert np.array_equal(r0, r1)


@pytest.mark.parametrize("r", [1, 4, 8, 16])
@pytest.mark.parametrize("layout", ["unaligned", "even", "pair", "aligned_forced"])
def test_async_mq_pass(r, layout, monkeypatch):
    """gc_psgd_mq_deferred_batched on layouts no single tensor map describes -- the cp.async feed
    (odd offsets; cols % 4 == 2 at offsets = 2 mod 4), the row-pair tensor maps (cols % 4 == 2,
    aligned offsets) -- and the cp.async feed forced on a TMA-capable layout: corrected =
    f32(g + r) written over the residuals bit for bit, nothing else touched, P = M Q within 1e-5
    of fp64, for a batch of T = 3 tensors x 2 workers."""
    import ctypes
    from paper_2407_01378_b200 import _native
    from paper_2407_01378_b200.configs import matrix_shape_for
    # unaligned: odd tensor offsets (4-byte copies); even: cols % 4 == 2 with even offsets (8-byte
    # copies, GPT-2's case); aligned_forced: a TMA-capable layout on the cp.async feed
    # pair: cols % 4 == 2 with 16-byte aligned tensor starts -> the row-pair tensor maps (ranks 4, 8, 16)
    d = {"unaligned": 150 * 150 - 7, "even": 150 * 150 - 8, "pair": 150 * 150 - 8,
         "aligned_forced": 200 * 200 - 8}[layout]
    rows, cols = matrix_shape_for(d)
    T, L = 3, 2
    pad = {"unaligned": 1, "even": 2, "pair": 4, "aligned_forced": 0}[layout]
    ld = T * (d + pad) + 3 * pad
    offs_t = [t * (d + pad) + pad for t in range(T)]
    row_offs = torch.tensor([w * ld + offs_t[t] for t in range(T) for w in range(L)], dtype=torch.int64,
                            device="cuda")
    if layout == "aligned_forced":
        monkeypatch.setenv("GC_PSGD_MQ_FEED", "async")
    g = torch.randn(L, ld, device="cuda")
    res = torch.randn(L, ld, device="cuda")
    q = torch.randn(T, cols, r, device="cuda")
    batch = _native.PsgdBatch(T, L, row_offs.data_ptr(), ld, None, 0, 0)
    hoffs = (ctypes.c_int64 * T)(*offs_t)
    lib = _native.lib()
    assert lib.gc_psgd_mq_deferred_supported(ctypes.byref(batch), hoffs, d, rows, cols, r, g.data_ptr(),
                                             res.data_ptr())
    assert bool(lib.gc_psgd_mq_tma_supported_batched(ctypes.byref(batch), hoffs, d, rows, cols, r, g.data_ptr(),
                                                     res.data_ptr())) == (layout == "aligned_forced")
    ws = torch.empty(int(lib.gc_psgd_workspace_bytes(T * L, rows, cols, r)), dtype=torch.uint8, device="cuda")
    p = torch.empty(T * L, rows, r, device="cuda")
    want_c = g + res
    r_before = res.clone()
    _native.call("gc_psgd_mq_deferred_batched", ctypes.byref(batch), hoffs, d, rows, cols, r, g.data_ptr(),
                 res.data_ptr(), q.data_ptr(), None, None, p.data_ptr(), ws.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    mask = torch.zeros(L, ld, dtype=torch.bool, device="cuda")
    for t in range(T):
        mask[:, offs_t[t]:offs_t[t] + d] = True
    assert torch.equal(res[mask], want_c[mask])             # corrected over the tensors
    assert torch.equal(res[~mask], r_before[~mask])         # nothing outside them touched
    for t in range(T):
        for w in range(L):
            m = torch.zeros(rows * cols, dtype=torch.float64, device="cuda")
            m[:d] = want_c[w, offs_t[t]:offs_t[t] + d].double()
            ref = m.reshape(rows, cols) @ q[t].double()
            got = p[t * L + w].double()
            assert (got - ref).abs().max().item() <= 1e-5 * ref.abs().max().item(), (t, w)   # the contract


@pytest.mark.parametrize("r", [1, 3, 4])
@pytest.mark.parametrize("layout", ["unaligned", "even", "pair", "aligned"])
def test_async_mtp_pass(r, layout, monkeypatch):
    """Q_w = M_w^T P_hat on a batch of T = 3 tensors with row offsets: gc_psgd_mtp (no host
    offsets: the cp.async-fed slabs, 16-, 8- or 4-byte copies by row alignment), the CUDA-core
    float4 / scalar pass (GC_PSGD_MTP=vec) and gc_psgd_mtp_batched (one tensor map per tensor when
    the rows are 16-byte aligned; row-pair maps when cols = 2 mod 4 and every tensor's P_hat rows are
    16-byte aligned -- "pair" at rank 4, the cp.async slabs at ranks 1 and 3) against fp64, all far
    inside the 1e-5 contract."""
    import ctypes
    from paper_2407_01378_b200 import _native
    from paper_2407_01378_b200.configs import matrix_shape_for
    d = {"unaligned": 150 * 150 - 7, "even": 150 * 150 - 8, "pair": 150 * 150 - 8, "aligned": 200 * 200 - 8}[layout]
    pad = {"unaligned": 1, "even": 2, "pair": 4, "aligned": 0}[layout]
    rows, cols = matrix_shape_for(d)
    T, L = 3, 2
    ld = T * (d + pad) + 3 * pad
    offs_t = [t * (d + pad) + pad for t in range(T)]
    row_offs = torch.tensor([w * ld + offs_t[t] for t in range(T) for w in range(L)], dtype=torch.int64,
                            device="cuda")
    c = torch.randn(L, ld, device="cuda")
    ph = torch.randn(T, rows, r, device="cuda")
    aligned = layout == "aligned"
    batch = _native.PsgdBatch(T, L, row_offs.data_ptr(), ld, None, 1 if aligned else 0, 0)
    lib = _native.lib()
    ws = torch.empty(int(lib.gc_psgd_workspace_bytes(T * L, rows, cols, r)), dtype=torch.uint8, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    outs = []
    hoffs = (ctypes.c_int64 * T)(*offs_t)
    for impl in ("", "vec", "batched"):   # batched: tensor maps per tensor when the rows allow (aligned)
        if impl == "vec":
            monkeypatch.setenv("GC_PSGD_MTP", impl)
        else:
            monkeypatch.delenv("GC_PSGD_MTP", raising=False)
        q = torch.empty(T * L, cols, r, device="cuda")
        if impl == "batched":
            _native.call("gc_psgd_mtp_batched", ctypes.byref(batch), hoffs, d, rows, cols, r, c.data_ptr(),
                         ph.data_ptr(), q.data_ptr(), ws.data_ptr(), sp)
        else:
            _native.call("gc_psgd_mtp", ctypes.byref(batch), d, rows, cols, r, c.data_ptr(), ph.data_ptr(),
                         q.data_ptr(), ws.data_ptr(), sp)
        outs.append(q)
    torch.cuda.synchronize()
    for t in range(T):
        for w in range(L):
            m = torch.zeros(rows * cols, dtype=torch.float64, device="cuda")
            m[:d] = c[w, offs_t[t]:offs_t[t] + d].double()
            ref = m.reshape(rows, cols).T @ ph[t].double()
            scale = ref.abs().max().item()
            for q in outs:
                assert (q[t * L + w].double() - ref).abs().max().item() <= 1e-6 * scale, (t, w)
