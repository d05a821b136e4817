import sys, numpy as np, torch
sys.path.insert(0,'.')
import oracle, paper_2309_06619_b200 as rt
from rtgen import configs
d=configs.config2(n=50001,gid0=777)
ctx=rt.Context(d['lexicon'],0)
lex=oracle.Lexicon(d['lexicon'])
dev=torch.device('cuda',0)
feat=ctx.score(torch.from_numpy(d['data']).to(dev), torch.from_numpy(d['offsets'].view(np.int32)).to(dev))
torch.cuda.synchronize()
g=feat.cpu().numpy().view(np.uint16); w=oracle.rule_gen(lex,d['data'],d['offsets'])
bad=np.nonzero((g!=w).any(1))[0]
print('bad',len(bad), 'tiles', sorted(set((bad//256).tolist()))[:20])
for i in bad[:8]:
    t=bytes(d['data'][d['offsets'][i]:d['offsets'][i+1]])
    print(i, i%256, g[i].tolist(), w[i].tolist(), t[:200])
