"""pytest plugin: run the reference package's OWN tests against the B200 GradientPipeline.

Test infrastructure, not product.  `tools/run_reference_tests.sh` stages an unmodified copy of
the reference (`pkg/src/gradcomp` and `pkg/tests`) under the git-ignored `baseline/_ref/` and runs

    PYTHONPATH=baseline/_ref/src:. python -m pytest baseline/_ref/tests/<file> -p tools.ref_shim.plugin

At start-up this plugin replaces `gradcomp.pipelines.GradientPipeline` -- the seam every pipeline
caller goes through (`make_pipeline`, `_one_shot` and so the `run_*_round` wrappers, the CLI;
pipelines.py:97-135, 418-472) -- with `RefSeamPipeline`: the reference's constructor signature, the
reference's config / SeedSpec objects converted field for field to this package's, and this
package's GradientPipeline (CUDA kernels on cuda:0) behind it.  Everything else the tests import
(compressor primitives used for hand simulations, collectives, transforms) stays the reference's.
A test that passes here exercises the drop-in exactly as a reference user would."""
from __future__ import annotations

import dataclasses


def _convert_config(cfg):
    import paper_2407_01378_b200 as gcb
    cls = getattr(gcb, type(cfg).__name__, None)
    if cls is None or not dataclasses.is_dataclass(cfg):
        return cfg   # not a config this package knows: the B200 pipeline raises TypeError as the reference does
    return cls(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(cfg)})


def _make_seam():
    import paper_2407_01378_b200 as gcb

    class RefSeamPipeline(gcb.GradientPipeline):
        """gradcomp.pipelines.GradientPipeline(config, num_workers, dim, seeds, error_feedback=None)."""

        def __init__(self, config, num_workers, dim, seeds, error_feedback=None):
            seeds = gcb.SeedSpec(int(seeds.experiment_seed)) if hasattr(seeds, "experiment_seed") else seeds
            super().__init__(_convert_config(config), num_workers, dim, seeds, error_feedback)

    return RefSeamPipeline


def pytest_configure(config):
    import gradcomp.pipelines as ref_pipelines
    ref_pipelines.GradientPipeline = _make_seam()
    config.addinivalue_line("markers", "b200_seam: reference tests run through the B200 GradientPipeline")


def pytest_report_header(config):
    import gradcomp.pipelines as ref_pipelines
    return f"gradcomp.pipelines.GradientPipeline -> {ref_pipelines.GradientPipeline.__mro__[1].__module__}" \
           f".{ref_pipelines.GradientPipeline.__mro__[1].__name__} (B200)"
