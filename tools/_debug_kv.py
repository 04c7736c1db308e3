import sys, torch
sys.path.insert(0, '.')
import torch.nn.functional as F
from paper_2402_13533_b200 import decoder, glue
from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder, _group_fwd
CFG = DecoderConfig(vocab=512, dim=256, heads=2, layers=2, ffn_dim=512, max_seq=64)
model = build_decoder(CFG, rank=8, bits=8, seed=3)
g = torch.Generator().manual_seed(11)
tokens = torch.randint(0, CFG.vocab, (2, CFG.max_seq), generator=g).cuda()
seq = tokens[0, :6].tolist()
l = len(seq)
rope = model.rope_tables(l, 'cuda')
x = model.embed[torch.tensor(seq, device='cuda')]
out, e = model.layers[0].forward(x, (1, l, CFG.heads), rope, keep=True)
cache = decoder.KvCache(model)
m = model.layers[0].mats
heads, d = CFG.heads, CFG.head_dim
for pos, t in enumerate(seq):
    cos, sin = cache.rope[0][pos:pos + 1], cache.rope[1][pos:pos + 1]
    xd = model.embed[int(t)].reshape(1, CFG.dim).contiguous()
    n1, _ = glue.rmsnorm(xd, model.layers[0].norm1)
    q, k, v = _group_fwd([m["wq"], m["wk"], m["wv"]], n1)
    qb = q.clone()
    glue.rope_(q, k, cos, sin, heads, 1)
    cache.k[0][pos].copy_(k[0]); cache.v[0][pos].copy_(v[0])
    keys = cache.k[0][:pos + 1].view(pos + 1, heads, d).transpose(0, 1)
    vals = cache.v[0][:pos + 1].view(pos + 1, heads, d).transpose(0, 1)
    ctx = F.scaled_dot_product_attention(q.view(heads, 1, d), keys, vals).reshape(1, CFG.dim)
    def rel(a, b): return float((a.float() - b.float()).abs().max() / b.float().abs().max())
    print(pos, 'norm1', rel(n1[0], e['norm1'][pos]), 'q', rel(q[0], e['q'][pos]), 'k', rel(k[0], e['k'][pos]), 'v', rel(v[0], e['v'][pos]), 'ctx', rel(ctx[0], e['ctx'][pos]))
