"""Print the GPU engine's 8B-shape output next to the oracle golden (tests/golden/llama8b_oracle.json):
token equality, out_hash equality and raw logit bits of steps 0 and 3.  python tools/llama8b_golden_check.py"""
import json, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2602_00182_b200.detcore import DecodePolicy, Engine
g = json.load(open('/root/repo/tests/golden/llama8b_oracle.json'))
eng = Engine(g["model"], "b200", max_batch=2, max_context=128)
for c in g["cases"]:
    prompt = np.array(c["prompt"], dtype=np.uint32)
    T = c["max_tokens"]
    pol = DecodePolicy.greedy(T) if c["kind"] == 0 else DecodePolicy.nucleus(c["p"], T)
    toks, logits, h = eng.generate([prompt], [pol], [c["seed"]])
    print("tokens", toks[0].tolist() == c["tokens"], "hash", h[0].hex() == c["out_hash"])
    print(" step0 gpu", [int(x) for x in logits[0][0, :8].view(np.uint32)])
    print(" step0 orc", c["logit_bits_step0_first8"])
    print(" last gpu", [int(x) for x in logits[0][-1, -8:].view(np.uint32)])
    print(" last orc", c["logit_bits_last_step_last8"])
