"""PyTorch DDP communication hook: the training-step caller of the compression path.

SURVEY.md §8(f) rank 2 / PAPER.md:117 ("implemented in NCCL and PyTorch DDP"): between the
backward pass and the optimizer step, every DDP gradient bucket is compressed, aggregated over
the ranks and decompressed by the B200 pipeline instead of DDP's all-reduce.  Each rank is one
reference worker (n = world size); every bucket keeps its own pipeline (EF residuals, warm Q),
keyed by the bucket index, and the round index advances once per optimizer step.

    from paper_2407_01378_b200.ddp import CompressionHookState, compression_hook
    state = CompressionHookState(RotatedQuantConfig(4, 8), SeedSpec(2024))
    ddp_model.register_comm_hook(state, compression_hook)

The hook's future resolves to the pipeline's estimate of the mean gradient (the reference's
RoundResult.estimate), identical on every rank.
"""

import torch
import torch.distributed as dist

from .distributed import DistributedGradientPipeline
from .vectors import SeedSpec


class CompressionHookState:
    def __init__(self, config, seeds: SeedSpec, *, group=None, validate: bool = False, record: bool = False):
        self.config = config
        self.seeds = seeds
        self.group = group
        self.validate = validate
        self.pipelines = {}
        self.round_index = 0
        self._seen: set[int] = set()
        self.last_results = {}
        self.record = record        # keep each bucket's input (tests / debugging)
        self.last_inputs = {}

    def pipeline_for(self, index: int, numel: int) -> DistributedGradientPipeline:
        pipe = self.pipelines.get(index)
        if pipe is None or pipe.dim != numel:
            world = dist.get_world_size(self.group)
            pipe = DistributedGradientPipeline(self.config, world, numel, self.seeds, group=self.group,
                                               validate=self.validate)
            self.pipelines[index] = pipe
        return pipe


def compression_hook(state: CompressionHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: bucket gradient -> compressed round -> mean-gradient estimate."""
    idx = bucket.index()
    if idx in state._seen:          # a bucket seen twice means a new optimizer step began
        state._seen.clear()
        state.round_index += 1
    state._seen.add(idx)
    buf = bucket.buffer()
    flat = buf.reshape(1, -1).to(torch.float32).contiguous()
    pipe = state.pipeline_for(idx, flat.numel())
    if state.record:
        state.last_inputs[idx] = flat.detach().clone()
    res = pipe.run_round(flat, state.round_index)
    state.last_results[idx] = res
    est = res.estimate_tensor.to(buf.dtype).reshape(buf.shape)
    fut = torch.futures.Future()
    fut.set_result(est)
    return fut
