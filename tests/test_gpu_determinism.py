"""Receipt determinism at scale (BASELINE configs 3 and 4, tiny model so it runs in seconds):
1000 and 10,000 replays of a nucleus-sampled request spread over batches, batch-size sweeps
1/8/64/256 and 1/4/8/6/10. The 8B shape: tools/determinism_sweep.py (profiles/determinism_r1.json)."""
import pytest

pytestmark = pytest.mark.gpu


def test_thousand_replays_and_batch_sweep():
    from paper_2602_00182_b200 import replicas
    from paper_2602_00182_b200.detcore import DecodePolicy, Engine

    eng = Engine("llama-tiny:replay", "b200", max_batch=256, max_context=128)
    V = eng.vocab
    p0 = replicas.synthetic_prompt(7, 24, V)
    pol = DecodePolicy.nucleus(0.9, 24)
    _, _, h = eng.generate([p0] * 1000, [pol] * 1000, [99] * 1000, batch_size=250, want_logits=False)
    assert len(set(h)) == 1
    prompts = [replicas.synthetic_prompt(i, 8 + i % 40, V) for i in range(256)]
    pols = [DecodePolicy.greedy(16) if i % 3 else DecodePolicy.nucleus(0.9, 16) for i in range(256)]
    seeds = [replicas.request_seed(i) for i in range(256)]
    ref = eng.generate(prompts, pols, seeds, batch_size=256, want_logits=False)[2]
    for bs in (64, 8, 1):
        assert eng.generate(prompts, pols, seeds, batch_size=bs, want_logits=False)[2] == ref, bs
    eng.close()


def test_ten_thousand_replays_tiny_match_oracle():
    """SPEC acceptance criterion 1 (10k-run determinism, reference SPEC.md:600): one nucleus request
    of the tiny model replayed 10,000 times in batches of 250 (and a batch-size grouping sweep
    1/4/8/6/10 as test_detcore.cpp:343-361): every out_hash identical, and equal to the CPU oracle's."""
    from oracle import oracle as O
    from paper_2602_00182_b200.detcore import DecodePolicy, Engine

    eng = Engine("llama-tiny:model-a", "b200", max_batch=250, max_context=128)
    g = O.Prng(31 ^ 0xABCD)
    prompt = [g.next_below(eng.vocab) for _ in range(20)]
    pol = DecodePolicy.nucleus(0.9, 24)
    _, _, h = eng.generate([prompt] * 10000, [pol] * 10000, [4242] * 10000, batch_size=250, want_logits=False)
    assert len(set(h)) == 1
    ot, ol = O.Llama("llama-tiny:model-a").generate(prompt, kind=2, p=0.9, max_tokens=24, seed=4242)
    assert h[0] == O.out_hash(ot, ol)
    prompts = [[(7 * i + j) % eng.vocab for j in range(3 + i % 17)] for i in range(40)]
    pols = [DecodePolicy.greedy(12) if i % 2 else DecodePolicy.nucleus(0.9, 12) for i in range(40)]
    seeds = list(range(40))
    ref = eng.generate(prompts, pols, seeds, batch_size=1, want_logits=False)[2]
    for bs in (4, 8, 6, 10):
        assert eng.generate(prompts, pols, seeds, batch_size=bs, want_logits=False)[2] == ref, bs
    eng.close()
