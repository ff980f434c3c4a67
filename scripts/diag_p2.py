import sys, numpy as np
sys.path.insert(0, '.')
import paper_2510_03996_b200 as fh
from oracle.ckks_oracle import Oracle
from tests.test_gpu_primitives import make_pair, _oracle_ct
for (logN, L, K, dnum, first, scale, special) in [(12, 24, 8, 3, 60, 50, 60), (16, 6, 2, 3, 50, 40, 60),
                                                  (12, 6, 2, 3, 60, 50, 60), (12, 24, 8, 3, 50, 40, 60),
                                                  (12, 12, 4, 3, 50, 40, 60), (12, 6, 4, 3, 50, 40, 60), (12, 9, 2, 3, 50, 40, 60)]:
    ctx, orc = make_pair(logN, L, K, dnum, first, scale, special, 7)
    rng = np.random.default_rng(1)
    vals, ct = _oracle_ct(orc, rng)
    g = orc.galois(1)
    key_ok = np.array_equal(ctx.download_key(g), orc.keygen(g))
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.keyswitch_raw(x, g, 1).words()
    ks0, ks1 = orc.keyswitch(ct[1], orc.keygen(g), 1)
    rs = np.array_equal(fh.rescale(x).words(), orc.rescale(ct))
    print((logN, L, K, first, scale), "key", key_ok, "ks0", np.array_equal(got[0], ks0), "ks1", np.array_equal(got[1], ks1),
          "rescale", rs, "limbs-bad", [i for i in range(L) if not np.array_equal(got[0][i], ks0[i])][:8], flush=True)
