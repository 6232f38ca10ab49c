"""Type-B RPCA (truncated nuclear norm, partial SVT) over
semi-online windows with basis transfer on the GPU against the
oracle's windowed driver (oracle/rpca.py rpca_windows): a video-shaped
synthetic input (the c3 recipe at a reduced frame size), windows of 5
frames, keep = 1, l = 3, eta = 2 (the paper's settings for n = 5)."""
import numpy as np
import pytest
import torch

from oracle.rpca import rpca_windows
from synth import make_config, omega
from tests.gpu_util import cm, np64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1509_00296_b200 as P
    return P


@pytest.mark.parametrize("transfer", [True, False])
def test_type_b_windows_against_oracle(P, transfer):
    H, W, frames, win, l, q, iters = 48, 64, 20, 5, 3, 2, 30
    cfg, d = make_config("c3", m=H * W, n=frames, H=H, W=W, nblocks=2, l=l, q=q, iters=iters)
    D = cm(d["D"], torch.float32)
    D64 = np64(D)
    ref = rpca_windows(D64, win, iters, l, q, lambda k: omega(cfg.seed, k, win, l).numpy(), keep=1,
                       rho=cfg.params["rho"], transfer=transfer)
    m = H * W
    h = P.Frsvt(m, win, l, q, rp=True, dtype=torch.float32, seed=cfg.seed)
    for w in range(frames // win):
        Dw = D[:, w * win:(w + 1) * win]
        E, A, L = torch.empty_like(Dw), torch.empty_like(Dw), torch.empty_like(Dw)
        st = h.rpca_state(Dw, E, A, L, rho=cfg.params["rho"], norm2_D=ref["windows"][w]["norm2"], keep=1,
                          transfer=transfer and w > 0)
        for k in range(iters):
            h.rpca_step(st, finalize=(k == iters - 1))
        Lr, Er = ref["windows"][w]["L"], ref["windows"][w]["E"]
        assert np.linalg.norm(np64(L) - Lr) <= 1e-3 * np.linalg.norm(Lr), w
        assert np.linalg.norm(np64(E) - Er) <= 1e-3 * max(np.linalg.norm(Er), 1e-3 * np.linalg.norm(D64)), w
        assert h.info().r == ref["windows"][w]["hist"]["r"][-1], w
