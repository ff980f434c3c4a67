for rb in 3 4; do FHEON_NTT_RB=$rb python -c "
import sys; sys.path.insert(0,'.')
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset('config2'))
for k in (0, 1, 3):
    b = 1 if k == 3 else 8
    ms = min(ctx.microbench(k, b, 24, 8, 10) for _ in range(3))
    print('rb $rb kind', k, 'ms per unit %.4f' % (ms / b))
"; done
FHEON_NTT_RB=4 timeout 600 python -m pytest tests/test_gpu_primitives.py -x -q -k "ntt or rotation" 2>&1 | tail -2
