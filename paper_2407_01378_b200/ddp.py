"""PyTorch DDP communication hook: the training-step caller of the compression path.

SURVEY.md §8(f) rank 2 / PAPER.md:117 ("implemented in NCCL and PyTorch DDP"): between the
backward pass and the optimizer step, every DDP gradient bucket is compressed, aggregated over
the ranks and decompressed by the B200 pipeline instead of DDP's all-reduce.  Each rank is one
reference worker (n = world size) and the round index advances once per optimizer step.

State is keyed by the bucket's parameter layout, not its index: DDP rebuilds its buckets after
the first iteration (and whenever the graph changes), so a bucket index can name a different
set of parameters from one step to the next.  Error-feedback residuals are per parameter: when a
layout appears for the first time, its pipeline starts from the residuals every parameter
carried in the layout it came from (the reference keeps a residual per coordinate,
pipelines.py:129-133, 168-170); the PowerSGD warm start (pipelines.py:366) is tied to the bucket's
matrix shape and restarts from a fresh seed matrix.  With `chunked=True` (PowerSGD) every parameter
is its own reference pipeline (DistributedTensorListPipeline: per-layer matrices, as PowerSGD is
used in practice); residuals carry over per parameter the same way.

A non-finite bucket (e.g. an fp16 GradScaler overflow step) is detected on every rank (the
pipeline's finite check is all-reduced), raises nothing inside autograd and leaves every
residual and warm Q untouched: the hook returns NaN gradients on all ranks so the scaler skips
the step everywhere, as the reference rejects non-finite gradients before any state changes
(pipelines.py:184-197).

    from paper_2407_01378_b200.ddp import CompressionHookState, compression_hook
    state = CompressionHookState(RotatedQuantConfig(4, 8), SeedSpec(2024))
    ddp_model.register_comm_hook(state, compression_hook)
"""

import torch
import torch.distributed as dist

from .configs import PowerSgdConfig
from .distributed import DistributedGradientPipeline, DistributedTensorListPipeline
from .vectors import SeedSpec


class CompressionHookState:
    def __init__(self, config, seeds: SeedSpec, *, group=None, validate: bool = True, record: bool = False,
                 chunked: bool = False):
        self.config = config
        # chunked=True with PowerSgdConfig: one reference pipeline per parameter (per-layer matrices,
        # the paper's and PyTorch's PowerSGD practice) instead of one matrix per bucket
        self.chunked = bool(chunked) and isinstance(config, PowerSgdConfig)
        self.seeds = seeds
        self.group = group
        self.validate = validate
        self.pipelines = {}          # layout key -> pipeline
        self.param_home = {}         # parameter id -> (layout key, offset, numel) of its residual
        self.round_index = 0
        self._seen: set[int] = set()
        self.last_results = {}
        self.skipped_rounds = []     # rounds whose bucket was non-finite (state untouched)
        self.record = record        # keep each bucket's input and layout (tests / debugging)
        self.last_inputs = {}
        self.last_layouts = {}

    @staticmethod
    def layout(bucket):
        """(parameter ids, offsets, numels) of a bucket: its gradients are packed in parameter order."""
        params = bucket.parameters()
        numels = [p.numel() for p in params]
        offs, o = [], 0
        for m in numels:
            offs.append(o)
            o += m
        if o != bucket.buffer().numel():
            raise ValueError("bucket buffer does not match its parameters' sizes")
        return tuple(id(p) for p in params), offs, numels

    def pipeline_for(self, bucket) -> DistributedGradientPipeline:
        ids, offs, numels = self.layout(bucket)
        key = ids
        pipe = self.pipelines.get(key)
        if pipe is not None:
            return pipe
        buf = bucket.buffer()
        world = dist.get_world_size(self.group)
        with torch.cuda.device(buf.device):
            if self.chunked:
                pipe = DistributedTensorListPipeline(self.config, world, numels, self.seeds, group=self.group,
                                                     device=buf.device, validate=self.validate)
            else:
                pipe = DistributedGradientPipeline(self.config, world, buf.numel(), self.seeds, group=self.group,
                                                   device=buf.device, validate=self.validate)
            if pipe.residuals_tensor is not None:   # carry every parameter's residual over
                dst = pipe.residuals_tensor[0]
                for pid, o, m in zip(ids, offs, numels):
                    home = self.param_home.get(pid)
                    if home is not None:
                        hk, ho, hm = home
                        src = self.pipelines[hk].residuals_tensor[0]
                        dst[o:o + m].copy_(src[ho:ho + hm])
        for pid, o, m in zip(ids, offs, numels):
            self.param_home[pid] = (key, o, m)
        self.pipelines[key] = pipe
        # layouts no parameter points at any more hold no live residuals
        live = {h[0] for h in self.param_home.values()}
        for k in [k for k in self.pipelines if k not in live]:
            del self.pipelines[k]
        return pipe


def compression_hook(state: CompressionHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: bucket gradient -> compressed round -> mean-gradient estimate."""
    idx = bucket.index()
    if idx in state._seen:          # a bucket seen twice means a new optimizer step began
        state._seen.clear()
        state.round_index += 1
    state._seen.add(idx)
    buf = bucket.buffer()
    pipe = state.pipeline_for(bucket)
    with torch.cuda.device(buf.device):
        flat = buf.reshape(1, -1).to(torch.float32).contiguous()
        if state.record:
            state.last_inputs[idx] = flat.detach().clone()
            state.last_layouts[idx] = state.layout(bucket)
        fut = torch.futures.Future()
        try:
            res = pipe.run_round(flat, state.round_index)
        except ValueError:          # non-finite on some rank: all ranks skip, EF state untouched
            state.skipped_rounds.append(state.round_index)
            fut.set_result(torch.full_like(buf, float("nan")))
            return fut
        state.last_results[idx] = res
        fut.set_result(res.estimate_tensor.to(buf.dtype).reshape(buf.shape))
    return fut
