for m in 0 1; do for k in 0 1 3 4; do FHEON_NTT_TWSMEM=$m python -c "
import sys; sys.path.insert(0,'.')
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset('config2'))
k=$k
b = 1 if k in (3,4) else 8
ms = min(ctx.microbench(k, b, 24, 8, 10) for _ in range(3))
print('mode $m kind', k, 'ms per unit', ms / b)
"; done; done
