"""Receipt v2: per-step Merkle roots of the logits in 4 KiB
leaves with the reference's DA tree rules, pinned by golden vectors generated from the reference's
own da.cpp (tests/golden/make_receipt_v2_golden.py). CPU: oracle and the product's host digest;
GPU: the digest kernel and the engine's DETGPU_F_RECEIPT_V2 path."""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "receipt_v2.json").read_text())


def _logits(seed, T, V):
    import importlib.util

    spec = importlib.util.spec_from_file_location("v2gold", Path(__file__).parent / "golden" / "make_receipt_v2_golden.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.logits(seed, T, V)


def test_oracle_matches_reference_merkle():
    from oracle import oracle as O

    assert O.merkle_root([]).hex() == GOLD["empty_root"]
    for c in GOLD["cases"]:
        lg = _logits(c["seed"], c["T"], c["V"])
        assert [O.step_root(lg[t]).hex() for t in range(c["T"])] == c["roots"], c["V"]
        assert O.hash_canonical_v2(c["tokens"], lg).hex() == c["out_hash_v2"]


def test_product_host_digest_matches_golden():
    from paper_2602_00182_b200._lib import lib
    from paper_2602_00182_b200.detcore import hash_canonical_v2

    for c in GOLD["cases"]:
        lg = np.ascontiguousarray(_logits(c["seed"], c["T"], c["V"]))
        for t in range(c["T"]):
            out = np.zeros(32, np.uint8)
            lib.detgpu_step_root(lg[t].ctypes.data, c["V"], out.ctypes.data)
            assert out.tobytes().hex() == c["roots"][t]
        assert hash_canonical_v2(c["tokens"], lg).hex() == c["out_hash_v2"]


def test_v2_differs_from_v1_and_sees_every_bit():
    from paper_2602_00182_b200.detcore import encode_canonical_output, hash_canonical_v2, sha256

    lg = _logits(11, 2, 5000)
    toks = [3, 4]
    h = hash_canonical_v2(toks, lg)
    assert h != sha256(encode_canonical_output(toks, lg))
    for t, v in [(0, 0), (1, 4999), (1, 1023), (0, 1024)]:
        lg2 = lg.copy()
        lg2.view(np.uint32)[t, v] ^= 1
        assert hash_canonical_v2(toks, lg2) != h
    assert hash_canonical_v2([3, 5], lg) != h


@pytest.mark.gpu
def test_gpu_step_roots_kernel_matches_golden():
    import torch
    from paper_2602_00182_b200._lib import check, lib

    for c in GOLD["cases"]:
        if c["T"] == 0:
            continue
        lg = torch.from_numpy(np.ascontiguousarray(_logits(c["seed"], c["T"], c["V"]))).cuda()
        roots = torch.zeros(c["T"] * 32, dtype=torch.uint8, device="cuda")
        check(lib.detgpu_k_step_roots(lg.data_ptr(), c["T"], c["V"], roots.data_ptr(), None))
        torch.cuda.synchronize()
        got = roots.cpu().numpy().reshape(c["T"], 32)
        assert [bytes(r).hex() for r in got] == c["roots"], c["V"]


@pytest.mark.gpu
@pytest.mark.parametrize("model,arch", [("llama-tiny:v2", "b200"), ("model-a", "archA")])
def test_engine_receipt_v2(model, arch):
    from oracle import oracle as O
    from paper_2602_00182_b200 import replicas
    from paper_2602_00182_b200.detcore import DecodePolicy, Engine

    eng = Engine(model, arch, max_batch=8, max_context=128 if arch == "b200" else 1)
    V = eng.vocab
    prompts = [replicas.synthetic_prompt(i, 8 + i, V) for i in range(5)]
    pols = [DecodePolicy.greedy(12), DecodePolicy.nucleus(0.9, 7), DecodePolicy.top_k(4, 3), DecodePolicy.greedy(0),
            DecodePolicy.greedy(1)]
    seeds = [replicas.request_seed(i) for i in range(5)]
    toks, logits, h1 = eng.generate(prompts, pols, seeds)
    toks2, logits2, h2 = eng.generate(prompts, pols, seeds, receipt_v2=True)
    _, nolog, h3 = eng.generate(prompts, pols, seeds, receipt_v2=True, want_logits=False, batch_size=2)
    for i in range(5):
        assert np.array_equal(toks[i], toks2[i]) and np.array_equal(logits[i].view(np.uint32), logits2[i].view(np.uint32))
        assert h2[i] == O.hash_canonical_v2(toks[i], logits[i]) == h3[i]
        assert h2[i] != h1[i]
    eng.close()
