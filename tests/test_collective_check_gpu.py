"""cli.py:436-573's collective-check on the real transport (paper_2407_01378_b200.collective_check):
every check passes over 1, 2 and 4 ranks (gloo with host staging, all ranks on the one B200), and an
injected wire width (inject_element_bits) makes the ring egress check fail, as in the reference."""
import pytest

from tests.dist_util import run_world
from tests.gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]


def _rank(rank, world, inject):
    import torch
    from paper_2407_01378_b200.collective_check import collective_check
    torch.cuda.set_device(0)
    return collective_check(2024, inject, device=torch.device("cuda", 0))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_collective_check_passes(world):
    out = run_world(_rank, world, (None,))
    for ok, lines in out:
        assert ok, "\n".join(lines)
        assert all(l.startswith("PASS") for l in lines)
        assert len(lines) == 17


def test_injected_wire_width_is_caught():
    out = run_world(_rank, 2, (16,))
    for ok, lines in out:
        assert not ok
        failed = [l for l in lines if l.startswith("FAIL")]
        assert len(failed) == 1 and "ring_egress_closed_form" in failed[0], lines
