"""Op-level GPU parity of individual sm_100a kernels through the C-ABI (the reference's
op-level tests, e.g. test_dstt.py:70-159, applied to our kernels)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_10466_b200 import _lib  # noqa: E402


def conv3x3_ref(x, w, b):
    """x (F,H,W,64) fp32, w (64,64,3,3), zero pad 1, LeakyReLU(0.2) -- dstt.py:241-242."""
    f, h, wd, c = x.shape
    xp = np.zeros((f, h + 2, wd + 2, c))
    xp[:, 1:-1, 1:-1] = x
    out = np.zeros((f, h, wd, w.shape[0]))
    for dy in range(3):
        for dx in range(3):
            out += xp[:, dy:dy + h, dx:dx + wd] @ w[:, :, dy, dx].T.astype(np.float64)
    out += b
    return np.where(out >= 0, out, 0.2 * out)


@pytest.mark.parametrize("shape", [(1, 2, 128), (2, 5, 200), (1, 64, 512)])
def test_tcgen05_conv3x3_vs_reference(shape):
    f, h, wd = shape
    rng = np.random.default_rng(7)
    x = rng.normal(0, 1, (f, h, wd, 64)).astype(np.float16)
    w = (rng.normal(0, 1, (64, 64, 3, 3)) * np.sqrt(2 / 576)).astype(np.float32)
    b = rng.normal(0, 0.1, 64).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    _lib.check(_lib.load().dr_op_conv3x3(f, h, wd, xd.data_ptr(), w.ctypes.data, b.ctypes.data,
                                         out.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream))
    got = out.float().cpu().numpy()
    ref = conv3x3_ref(x.astype(np.float64), w.astype(np.float16).astype(np.float64), b)
    err = np.abs(got - ref)
    assert err.max() < 1e-2 + 2e-3 * np.abs(ref).max(), err.max()


_SPLIT_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[2])
from paper_2509_10466_b200 import DsttConfig, DsttEngine, synth
cfg = DsttConfig.baseline(256, mask_dilate=2, mask_feather_sigma=1.0)
eng = DsttEngine(cfg, seed=0)
imgs, masks = synth.frame_pool("C1", 2, size=256)
rng = np.random.default_rng(1)
slots = [torch.from_numpy(rng.normal(0, 1, (2, cfg.tokens, 64)).astype(np.float32)).cuda()
         for _ in range(2)]
res = eng.run(torch.from_numpy(imgs).cuda(), torch.from_numpy(masks).cuda(), slots)
np.save(sys.argv[1], res["fill"].cpu().numpy() if "fill" in res else res["out"].cpu().numpy())
"""


def test_attention_key_split_one_two_four_agree(tmp_path):
    """The per-launch key split (attention_ksplit: 1 CTA per query-tile group at large
    batch, clusters of 2 or 4 merged through DSMEM at small batch) must not change the
    result beyond fp32 merge rounding."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    repo = str(Path(__file__).resolve().parents[1])
    outs = []
    for k in (1, 2, 4):
        dst = tmp_path / f"k{k}.npy"
        subprocess.run([sys.executable, "-c", _SPLIT_SCRIPT, str(dst), repo], check=True,
                       env={**os.environ, "DR_ATTN_KSPLIT": str(k)}, timeout=300)
        outs.append(np.load(dst))
    for o in outs[1:]:
        assert outs[0].shape == o.shape
        assert np.abs(outs[0].astype(np.float64) - o).max() <= 2e-3
