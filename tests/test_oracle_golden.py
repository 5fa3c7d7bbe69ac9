"""Pin the CPU oracle (oracle/gradcomp_oracle.py) against golden vectors from the reference."""
import numpy as np
import pytest

from oracle import gradcomp_oracle as orc
from tests.golden_util import CASES, EXACT_SCHEMES, load, seeds


def test_seed_chain_matches_reference():
    s = seeds()
    for k, v in s["splitmix64"].items():
        assert orc.splitmix64(int(k)) == v
    for k, v in s["fnv1a64"].items():
        assert orc.fnv1a64(k) == v
    for entry, pcg in zip(s["stream_seed"], s["pcg"]):
        seed = orc.stream_seed(2024, entry["tag"], entry["round"], entry["worker"])
        assert seed == entry["seed"]
        st, inc = orc.pcg64_state_from_seed(seed)
        assert (st, inc) == (pcg["state"], pcg["inc"])
        draws = []
        for _ in range(5):
            st, u = orc.pcg64_next(st, inc)
            draws.append((u >> 11) * 2.0 ** -53)
        assert draws == pcg["random5"]
        # integers(0, 2): top bit of the low then high u32 half of each output
        st, inc = orc.pcg64_state_from_seed(seed)
        bits = []
        for _ in range(32):
            st, u = orc.pcg64_next(st, inc)
            bits += [(u & 0xFFFFFFFF) >> 31, u >> 63]
        assert bits == pcg["bits64"]


def test_chunk_norms_pairwise_order():
    with np.load(f"{__import__('tests.golden_util', fromlist=['GOLDEN']).GOLDEN}/chunk_norms.npz") as z:
        for C in (1, 3, 8, 9, 64, 100, 129, 1000):
            v, ref = z[f"v_{C}"], z[f"norms_{C}"]
            assert np.array_equal(orc.chunk_sq_norms(v, C), ref)
            # the scalar restatement of numpy's pairwise order is bit-identical too
            buf = np.zeros(ref.size * C)
            buf[: v.size] = v
            sq = buf.reshape(-1, C) ** 2
            assert [orc.pairwise_sum(list(r)) for r in sq] == list(ref)


@pytest.mark.parametrize("name", ["thc_steps_a", "thc_steps_b", "thc_steps_c"])
def test_thc_intermediates(name):
    meta, a = load(name)
    n, d, seed, r = meta["n"], meta["d"], meta["seed"], meta["round"]
    corrected = list(a["corrected"])
    out = orc.thc_round(corrected, seed, r, meta["q"], meta["b"], meta["max_block"])
    assert out["block"] == meta["block"] and out["padded"] == meta["padded"]
    assert np.array_equal(out["signs"], a["signs"])
    assert np.array_equal(np.stack(out["rotated"]), a["rotated"])
    assert np.array_equal(out["shared"], a["shared"])
    assert np.array_equal(np.stack(out["codes"]), a["codes"])
    assert np.array_equal(out["sums"], a["sums"])
    assert out["clip_events"] == meta["clip_events"] and out["total_adds"] == meta["total_adds"]
    assert np.array_equal(out["estimate"], a["estimate"])
    assert np.array_equal(np.stack(out["own"]), a["own"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_rounds_match_reference(name):
    scheme, params = CASES[name]
    meta, a = load(name)
    n, d, seed = meta["n"], meta["d"], meta["seed"]
    ef = meta["error_feedback"]
    state = orc.OracleState([np.zeros(d, np.float32) for _ in range(n)] if ef else None)
    for st in meta["stats"]:
        r = st["round"]
        out = orc.run_round(scheme, params, state, list(a[f"grads_{r}"]), seed, r)
        if scheme in EXACT_SCHEMES:
            assert np.array_equal(out["estimate"], a[f"estimate_{r}"])
            if ef:
                assert np.array_equal(np.stack(state.residuals), a[f"residuals_{r}"])
        else:
            np.testing.assert_allclose(out["estimate"], a[f"estimate_{r}"], rtol=1e-5, atol=1e-6)
            if ef:
                np.testing.assert_allclose(np.stack(state.residuals), a[f"residuals_{r}"], rtol=1e-5, atol=1e-5)
        assert out["input_bits"] / d == pytest.approx(st["input_bits_per_coord"], rel=1e-12)
        assert out["nmse"] == pytest.approx(st["nmse"], rel=1e-9, abs=1e-12)
        if scheme == "rotated_quant":
            assert out["clip_events"] == st["clip_events"]
            assert out["total_adds"] == st["total_adds"]
            assert out["range_clips"] == st["range_clips"]
            assert out["code_sigma"] == pytest.approx(st["code_sigma"], rel=1e-12)
