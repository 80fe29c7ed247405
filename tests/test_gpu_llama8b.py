"""BASELINE.json configs[1], [2] and [3] at the Llama-3-8B shape, pinned to the CPU oracle.

tests/golden/llama8b_bench_oracle.json holds the oracle's output (tests/golden/
make_llama8b_bench_golden.py) for bench.py's own workload: model "llama3-8b:bench", request 0
(synthetic prompt of 512 tokens, greedy 256) and request 1 (512 tokens, nucleus p = 0.9, 256).
These tests check the GPU engine against it:

* cfg 2: request 0 at batch 1 -- tokens, logit bits of four steps, every step's logits SHA-256,
  out_hash (the reference receipt) and the receipt v2 digest equal the oracle's;
* cfg 3: 256 distinct requests (requests 0 and 1 plus 254 with ragged prompts 16..512 and mixed
  greedy / top-k / nucleus policies) at batch 1, 6, 8, 10, 51, 64, 77, 205, 256 (the
  reference's batch-grouping sweep, test_detcore.cpp:343-361, with +-20 % perturbations of
  8 / 64 / 256) and in reversed order: every receipt identical, and requests 0 / 1
  inside a batch of 256 (streamed attention, many-column GEMM epilogues) equal the oracle;
* cfg 4: request 1 replayed 1,000 times (4 batches of 250, receipt v2 on the GPU) plus 8 single
  replays (reference receipt): all equal the oracle's digests.
"""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden" / "llama8b_bench_oracle.json"


def _golden():
    g = json.loads(GOLDEN.read_text())
    return g, {c["name"]: c for c in g["cases"]}


def _policy(c):
    from paper_2602_00182_b200.detcore import DecodePolicy

    return DecodePolicy.greedy(c["max_tokens"]) if c["kind"] == 0 else DecodePolicy.nucleus(c["p"], c["max_tokens"])


def _request(c, V):
    from paper_2602_00182_b200 import replicas

    pr = replicas.synthetic_prompt(c["request_index"], c["prompt_len"], V)
    import hashlib

    assert hashlib.sha256(pr.astype("<u4").tobytes()).hexdigest() == c["prompt_sha256"]
    return pr, _policy(c), c["seed"]


@pytest.fixture(scope="module")
def eng8b():
    from paper_2602_00182_b200.detcore import Engine

    g, _ = _golden()
    eng = Engine(g["model"], "b200", max_batch=256, max_context=768)
    yield eng
    eng.close()


def test_bench_request_matches_oracle_batch1(eng8b):
    import hashlib

    _, cases = _golden()
    c = cases["greedy"]
    pr, pol, seed = _request(c, eng8b.vocab)
    toks, logits, hashes = eng8b.generate([pr], [pol], [seed], batch_size=1)
    lg = logits[0]
    assert toks[0].tolist() == c["tokens"]
    step_sha = [hashlib.sha256(lg[t].astype("<f4").tobytes()).hexdigest() for t in range(lg.shape[0])]
    bad = [t for t in range(len(step_sha)) if step_sha[t] != c["step_logits_sha256"][t]]
    assert not bad, f"logits differ from the oracle from step {bad[0]} on ({len(bad)} steps)"
    for t, bits in c["logit_bits"].items():
        t = int(t)
        got = [int(x) for x in lg[t, :8].view(np.uint32)] + [int(x) for x in lg[t, -8:].view(np.uint32)]
        assert got == bits, t
    assert hashes[0].hex() == c["out_hash"]
    _, _, h2 = eng8b.generate([pr], [pol], [seed], batch_size=1, want_logits=False, receipt_v2=True)
    assert h2[0].hex() == c["out_hash_v2"]


def test_batch_invariance_sweep_256_requests(eng8b):
    from paper_2602_00182_b200 import replicas
    from paper_2602_00182_b200.detcore import DecodePolicy

    _, cases = _golden()
    V = eng8b.vocab
    prompts, pols, seeds = [], [], []
    for name in ("greedy", "nucleus"):
        pr, pol, sd = _request(cases[name], V)
        prompts.append(pr)
        pols.append(pol)
        seeds.append(sd)
    for i in range(2, 256):
        prompts.append(replicas.synthetic_prompt(i, 16 + (i * 53) % 497, V))
        T = 8 + (i * 7) % 41
        pols.append([DecodePolicy.greedy(T), DecodePolicy.nucleus(0.9, T), DecodePolicy.top_k(50, T)][i % 3])
        seeds.append(replicas.request_seed(i))
    ref = eng8b.generate(prompts, pols, seeds, batch_size=256, want_logits=False)[2]
    assert ref[0].hex() == cases["greedy"]["out_hash"]
    assert ref[1].hex() == cases["nucleus"]["out_hash"]
    assert len(set(ref)) == 256
    for bs in (205, 77, 64, 51, 10, 8, 6, 1):
        h = eng8b.generate(prompts, pols, seeds, batch_size=bs, want_logits=False)[2]
        bad = [i for i in range(256) if h[i] != ref[i]]
        assert not bad, (bs, bad[:8])
    rev = list(range(256))[::-1]
    hr = eng8b.generate([prompts[i] for i in rev], [pols[i] for i in rev], [seeds[i] for i in rev], batch_size=64,
                        want_logits=False)[2]
    assert [hr[rev.index(i)] for i in range(256)] == ref


def test_nucleus_thousand_replays_match_oracle(eng8b):
    _, cases = _golden()
    c = cases["nucleus"]
    pr, pol, seed = _request(c, eng8b.vocab)
    n = 1000
    _, _, hv2 = eng8b.generate([pr] * n, [pol] * n, [seed] * n, batch_size=250, want_logits=False, receipt_v2=True)
    assert len(hv2) == n and set(h.hex() for h in hv2) == {c["out_hash_v2"]}
    for _ in range(8):
        toks, _, h = eng8b.generate([pr], [pol], [seed], batch_size=1, want_logits=False)
        assert h[0].hex() == c["out_hash"]
        assert toks[0].tolist() == c["tokens"]


def test_decode_graph_stress_batch_transitions(eng8b):
    """Regression for the streamed-attention ring's phase-parity ABA (fixed in round 2: a consumer
    group waiting for a stage's second use while the first use was still in flight passed its
    parity wait early and the ring deadlocked; the mbarrier watchdog trapped ~1 % of batch-256
    sweeps). CUDA-graph decode steps at batch 1 / 8 / 64 / 256, 20 rounds: every launch succeeds."""
    import ctypes as C

    from paper_2602_00182_b200 import _lib as L

    for _ in range(20):
        for b in (1, 8, 64, 256):
            ms = C.c_float()
            L.check(L.lib.detgpu_profile_graph(eng8b.h, b, 640, 0, 10, C.byref(ms)), eng8b.h)
