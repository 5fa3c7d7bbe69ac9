"""Loading helpers for the golden fixtures written by tests/golden/make_golden.py."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        arrs = {k: z[k] for k in z.files if k != "meta"}
        meta = json.loads(str(z["meta"]))
    return meta, arrs


def seeds():
    with open(os.path.join(GOLDEN, "seeds.json")) as f:
        return json.load(f)


# (scheme, params) for each whole-round fixture, mirroring make_golden.py
CASES = {
    "thc_a": ("rotated_quant", dict(quant_bits=4, wire_bits=4, rotation_block=256)),
    "thc_b": ("rotated_quant", dict(quant_bits=4, wire_bits=8, rotation_block=1024)),
    "thc_c": ("rotated_quant", dict(quant_bits=3, wire_bits=5, rotation_block=1024)),
    "thc_d": ("rotated_quant", dict(quant_bits=4, wire_bits=4, rotation_block=1 << 15)),
    "thc_e": ("rotated_quant", dict(quant_bits=8, wire_bits=16, rotation_block=64)),
    "thc_f": ("rotated_quant", dict(quant_bits=2, wire_bits=2, rotation_block=2)),
    "topk_a": ("topk", dict(k=50)),
    "topk_b": ("topk", dict(k=7)),
    "chunked_a": ("chunked_topk", dict(chunk_size=64, chunks_selected=10)),
    "chunked_b": ("chunked_topk", dict(chunk_size=16, chunks_selected=20, permute=True)),
    "chunked_c": ("chunked_topk", dict(chunk_size=7, chunks_selected=5)),
    "psgd_a": ("powersgd", dict(rank=4)),
    "psgd_b": ("powersgd", dict(rank=2)),
    "psgd_c": ("powersgd", dict(rank=2, warm_start=False)),
    "dense16": ("dense", dict(bits=16)),
    "dense32": ("dense", dict(bits=32)),
}
EXACT_SCHEMES = {"rotated_quant", "topk", "chunked_topk", "dense"}
