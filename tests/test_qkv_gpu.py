"""K6 (csrc/qkv_proj.cu): the tcgen05 QKV projection, and its fused
sequence-parallel scatter, on one B200."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2511_23113_b200 as D
from paper_2511_23113_b200.qkv import QkvScatter, qkv_project
from paper_2511_23113_b200.sp import home_range, rank_layouts

pytestmark = pytest.mark.gpu


def _inputs(T, C, H, d, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(T, C, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(3 * H * d, C, generator=g) / C ** 0.5).to(torch.bfloat16).cuda()
    b = (torch.randn(3 * H * d, generator=g) * 0.1).to(torch.bfloat16).cuda()
    return x, w, b


@pytest.mark.parametrize("T,C,H,d", [(512, 1024, 8, 128), (448, 512, 4, 64), (1000, 640, 2, 128)])
def test_qkv_project_matches_fp32_reference(T, C, H, d):
    x, w, b = _inputs(T, C, H, d, 1)
    y = qkv_project(x, w, H, d, bias=b)
    ref = x.float() @ w.float().T + b.float()
    torch.cuda.synchronize()
    err = (y.float() - ref).abs().max().item()
    rel = ((y.float() - ref).norm() / ref.norm()).item()
    assert err <= 3e-2 and rel <= 1e-2, (err, rel)


@pytest.mark.parametrize("strategy", ["U8R1", "U4R2", "U2R4", "U1R8"])
@pytest.mark.parametrize("balanced", [False, True])
def test_fused_qkv_scatter_equals_projection_then_exchange(strategy, balanced):
    # Every home rank's projection stores its rows straight into the
    # consuming ranks' local Q/K/V buffers; the result equals projecting home
    # and then moving the rows as the all-to-all(v) of sp.py would.
    H, d, C, S = 16, 128, 512, 4096
    nb = S // 64
    st = D.parse_strategy(strategy)
    G = st.gpus()
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 41))
    plan = D.plan_dual(masks, st).plan if balanced else D.default_plan(masks, st)
    lays = rank_layouts(st, plan, nb, nb)
    x, w, b = _inputs(S, C, H, d, 2)
    dev = x.device
    qbuf = [torch.zeros(len(l.q_blocks) * 64, len(l.heads), d, device=dev, dtype=torch.bfloat16) for l in lays]
    kbuf = [torch.zeros(len(l.kv_groups[l.r]) * 64, len(l.heads), d, device=dev, dtype=torch.bfloat16) for l in lays]
    vbuf = [torch.zeros_like(t) for t in kbuf]
    Y = torch.empty(S, 3 * H * d, device=dev, dtype=torch.bfloat16)
    for g in range(G):
        lo, hi = home_range(g, G, nb)
        xh = x[lo * 64:hi * 64].contiguous()
        Y[lo * 64:hi * 64] = qkv_project(xh, w, H, d, bias=b)
        sc = QkvScatter(lays, g, nb, [t.data_ptr() for t in qbuf], [t.data_ptr() for t in kbuf],
                        [t.data_ptr() for t in vbuf], dev)
        qkv_project(xh, w, H, d, bias=b, scatter=sc)
    torch.cuda.synchronize()
    Y = Y.view(S, 3, H, d)
    rows = lambda blocks: torch.as_tensor(np.concatenate([np.arange(b * 64, b * 64 + 64) for b in blocks])
                                          if len(blocks) else np.zeros(0, np.int64), device=dev)
    for l in lays:
        hs = torch.as_tensor(l.heads, device=dev)
        assert torch.equal(qbuf[l.rank], Y[rows(l.q_blocks)][:, 0][:, hs])
        kv = rows(l.kv_groups[l.r])
        assert torch.equal(kbuf[l.rank], Y[kv][:, 1][:, hs])
        assert torch.equal(vbuf[l.rank], Y[kv][:, 2][:, hs])
