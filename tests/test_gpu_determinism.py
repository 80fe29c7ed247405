"""Receipt determinism at scale (BASELINE configs 3 and 4, tiny model so it runs in seconds):
1000 replays of a nucleus-sampled request spread over batches, and a batch-size sweep 1/8/64/256."""
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
