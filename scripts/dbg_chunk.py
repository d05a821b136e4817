"""Debug: the random-runs chunk-boundary case of tests/test_gpu_parity.py, first failing requests."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, rtgen
import paper_2309_06619_b200 as rt
from rtgen import configs
rng = np.random.default_rng(23)
stems = ["history", "stuff", "bank", "john", "what", "why", "and", "or", "flies", "like", "art", "poverty",
         "x" * 14, "y" * 16, "z" * 20, "abcdefghijklmnopqrstuvwxyzabcdefghij", "a"]
tails = ["", "s", "es", "ed", "ing", "'s", "n't", "'ll", "'re", "'ve", "'m", "'d", "s's", "ing's"]
t = []
for _ in range(96 * 32):
    parts = []
    for _ in range(int(rng.integers(1, 40))):
        w = rng.choice(stems) + rng.choice(tails)
        if rng.random() < 0.1:
            w = w.upper()
        if rng.random() < 0.05:
            w = w * int(rng.integers(2, 5))
        parts.append(w)
        parts.append(rng.choice([" ", "  ", ", ", ". ", "? ", "", "\t"]))
    t.append("".join(parts)[: int(rng.integers(0, 400))])
if len(sys.argv) > 1:
    t = t[:int(sys.argv[1])]
data, off = rtgen.pack_texts(t)
lex = oracle.Lexicon(configs.read_lexicon())
ctx = rt.Context(configs.read_lexicon(), 0)
dev = torch.device("cuda", 0)
feat = ctx.score(torch.from_numpy(data).to(dev), torch.from_numpy(off.view(np.int32)).to(dev))
torch.cuda.synchronize()
got = feat.cpu().numpy().view(np.uint16)
want = oracle.rule_gen(lex, data, off)
bad = np.nonzero((got != want).any(1))[0]
print("requests", len(t), "bad", len(bad))
for i in bad[:6]:
    print(i, off[i], off[i + 1], bytes(data[off[i]:off[i + 1]]))
    print("   got ", got[i].tolist())
    print("   want", want[i].tolist())
