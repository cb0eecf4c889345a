"""The programmatic-dependent-launch chain (K1a -> K1b -> K2, SAB_PDL) changes only when
kernels start, never what they compute: outputs and K1 codes with PDL on and off must be
bit-identical.  Each arm runs in its own process because the library reads SAB_PDL once."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = r"""
import hashlib, torch
from paper_2410_02367_b200 import sageattn, synth
h = hashlib.sha256()
for (u, n, d, causal) in [(4, 2048, 128, True), (3, 1000, 64, False), (2, 4133, 128, False)]:
    q, k, v = (torch.from_numpy(synth.tensor(s, (u, n, d))).reshape(1, u, n, d).cuda() for s in (1, 2, 3))
    o = sageattn.sage_attention_cuda(q, k, v, causal=causal)
    torch.cuda.synchronize()
    h.update(o.cpu().numpy().tobytes())
print(h.hexdigest())
"""


def _run(pdl: str) -> str:
    env = dict(os.environ, SAB_PDL=pdl)
    r = subprocess.run([sys.executable, "-c", _SNIPPET], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_pdl_on_off_bit_identical():
    on, off = _run("1"), _run("0")
    assert len(on) == 64 and on == off
