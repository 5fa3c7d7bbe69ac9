"""Helpers shared by the GPU parity tests."""
import numpy as np
import pytest
import torch

from oracle import gradcomp_oracle as orc
from tests.golden_util import CASES, load

needs_gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def config_for(scheme, params):
    import paper_2407_01378_b200 as gcb
    if scheme == "rotated_quant":
        return gcb.RotatedQuantConfig(params["quant_bits"], params["wire_bits"], params.get("rotation_block", 1024))
    if scheme == "topk":
        return gcb.TopKConfig(params["k"])
    if scheme == "chunked_topk":
        return gcb.ChunkedTopKConfig(params["chunk_size"], params["chunks_selected"], params.get("permute", False))
    if scheme == "powersgd":
        return gcb.PowerSgdConfig(params["rank"], params.get("warm_start", True), params.get("bypass_below", 4096))
    return gcb.DenseConfig(params["bits"])


def run_golden_case(name, **pipe_kw):
    """Run a golden fixture through GradientPipeline; yield (round stats, result, pipe, arrays)."""
    import paper_2407_01378_b200 as gcb
    scheme, params = CASES[name]
    meta, a = load(name)
    pipe = gcb.make_pipeline(config_for(scheme, params), meta["n"], meta["d"], gcb.SeedSpec(meta["seed"]),
                             None if meta["error_feedback"] else False, **pipe_kw)
    for st in meta["stats"]:
        r = st["round"]
        res = pipe.run_round(list(a[f"grads_{r}"]), r)
        yield st, res, pipe, a


def oracle_rounds(scheme, params, grads_per_round, seed, ef=True):
    n, d = len(grads_per_round[0]), grads_per_round[0][0].size
    state = orc.OracleState([np.zeros(d, np.float32) for _ in range(n)] if ef else None)
    outs = []
    for r, grads in enumerate(grads_per_round):
        out = orc.run_round(scheme, params, state, grads, seed, r)
        out["residuals"] = None if state.residuals is None else [x.copy() for x in state.residuals]
        outs.append(out)
    return outs
