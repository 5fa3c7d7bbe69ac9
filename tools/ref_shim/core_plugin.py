"""pytest plugin: the reference's GradientPipeline with only its THC scheme core swapped for the
C-ABI binding of tools/ref_shim/round_quant_core.py.  The reference keeps its
own run_round, EF bookkeeping, ledger and RoundResult; `_round_quant` (pipelines.py:260-322) runs
on the B200 kernels through ctypes.  `bash tools/run_reference_tests.sh run-core`."""


def pytest_configure(config):
    import gradcomp.pipelines as ref_pipelines

    from tools.ref_shim.round_quant_core import round_quant_b200

    def _round_quant(self, corrected, ledger, round_index):
        return round_quant_b200(self, corrected, ledger, round_index)

    ref_pipelines.GradientPipeline._round_quant = _round_quant


def pytest_report_header(config):
    return "gradcomp.pipelines.GradientPipeline._round_quant -> tools.ref_shim.round_quant_core (ctypes, B200)"
