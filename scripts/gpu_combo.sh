# (batches in flight) x (images per batch) sweep of the ResNet-20 forward (scripts/ab_batch.py)
set -x
FLIGHT=2 timeout 600 python scripts/ab_batch.py 4 6 2>&1 | grep -E "in.flight"
FLIGHT=3 timeout 600 python scripts/ab_batch.py 2 3 2>&1 | grep -E "in.flight"
FLIGHT=4 timeout 600 python scripts/ab_batch.py 2 3 2>&1 | grep -E "in.flight"
FLIGHT=1 timeout 600 python scripts/ab_batch.py 4 8 2>&1 | grep -E "in.flight"
