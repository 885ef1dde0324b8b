import numpy as np, sys
sys.path.insert(0, '.')
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen, pcpqidx
from oracle.oracle import Port, Ref
cfg = datagen.CONFIGS['c1']
data = datagen.synth_index(cfg, seed=1, n=20000)
Q = datagen.queries(cfg, 3, seed=2).numpy()
idx = P.deserialize(data)
pi = Port().parse(data)
ri = Ref().open(data) if Ref.available() else None
ix = pcpqidx.deserialize(data)
for qi in range(3):
    got = P.score_query(idx, Q[qi]); want, _ = pi.score_query(Q[qi])
    bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
    print('query', qi, 'mismatches', len(bad), bad[:10])
    if ri is not None:
        rw, _ = ri.score_query(Q[qi]); print(' ref==port', rw.tobytes() == want.tobytes())
    for i in bad[:3]:
        print('  pt', i, got[i], want[i], ix.center_codes[i], ix.scalar_codes[i])
        # recompute in numpy float32 sequentially
        eta, etal, _ = pi.build_lut(Q[qi])
        acc = np.float32(-0.0)
        for j in range(cfg.m):
            t = np.float32(eta[j*16 + ix.center_codes[i, j]]) * np.float32(ix.scalar_codebooks[j, ix.scalar_codes[i, j]])
            acc = np.float32(acc + np.float32(t))
        print('  numpy', acc)
    # batch score_all as well
    g2 = P.score_all_batch(idx, Q)
    print(' batch mismatches', [(g2[b].view(np.uint32) != pi.score_query(Q[b])[0].view(np.uint32)).sum() for b in range(3)])
lut = P.build_lookup_table(idx, Q[0]); e2, l2, _ = pi.build_lut(Q[0])
print('lut eta eq', lut.eta.tobytes() == e2.tobytes(), 'etal eq', lut.eta_lambda.tobytes() == l2.tobytes())
