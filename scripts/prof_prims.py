"""Small driver for ncu captures of individual primitives (config-2 sizes)."""
import sys
sys.path.insert(0, '.')
import paper_2510_03996_b200 as fh
kind = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ctx = fh.SlotContext(fh.ContextConfig.preset("config2"))
print(kind, ctx.microbench(kind, 8 if kind not in (3, 4) else 1, 24, 8, 3))
