"""The drop-in seam, end to end: the reference's OWN acceptance harness
(/root/reference/proj/tests/acceptance.cpp, compiled unchanged with its layers,
Chebyshev evaluator, packing, key planner, model builder and runtime) linked
against integration/backend_b200.cpp -- the reference's backend API
(backend.hpp:134-153) implemented on the B200 engine's C ABI -- instead of the
reference's cleartext simulator (backend.cpp).  Every SlotVector is an RNS-CKKS
ciphertext in HBM; every rotate / mult / bootstrap runs the sm_100a kernels.

Criteria and their own tolerances (acceptance.cpp:1-18): 1 randomized layer
equivalence vs the dense oracle within 1e-9; 2 special 3x3 == pad + generic
(1e-9); 3 both striding flavours (1e-9); 4 key counts; 5 degree-59 activation
within the frozen bound and 1e-8 of the direct sum; 6 output-width formula; 7
LeNet-shaped model argmax >= 99/100 in <= 300 s; 9 lazy weights / block keys
bit-identical; 10 depth ledger.  Criterion 8 needs MNIST (SKIP by design).
Built by integration/Makefile (from /root/reference, in the build container);
the binary and integration/_build/refdata travel to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 6, 7, 9, 10])
def test_reference_acceptance_on_b200_backend(criterion):
    if not os.path.exists(BIN):
        pytest.fail("integration/_build/acceptance_b200 not built (make -C integration)")
    r = subprocess.run([BIN, str(criterion)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and f"[PASS] criterion {criterion}" in out, out[-2000:]
