"""PyTorch module API (paper_2605_17633_b200.modules) on the B200 (marker: gpu).

  * the module tree has SAM's ImageEncoderViT parameter names, and a state_dict round trip
    reproduces the output bit for bit; an in-place parameter update invalidates the cache;
  * at density = keep_fraction = 1 the SparseSAM encoder computes SAM's dense encoder: checked
    against dense.DenseSAMEncoder (torch / cuBLAS / SDPA, the same weights) with the encoder
    tolerance of tests/test_gpu_encoder.py (cosine >= 0.999, rel-Frobenius <= 3e-2);
  * SparseSAMBlock standalone == the one-block engine; StripeSortAttention at density 0.4 vs the
    float64 masked oracle on the module's own projections; ResidualConsistencyMLP vs torch.
"""

import pytest

from oracle import zs_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import torch.nn.functional as F

    from paper_2605_17633_b200 import modules as M
    from paper_2605_17633_b200.dense import DenseSAMEncoder
    from paper_2605_17633_b200.encoder import StripeSortEncoder


@pytest.fixture(autouse=True)
def _no_grad():
    """Inference-only module API: the reference math runs without autograd too."""
    with torch.no_grad():
        yield


def _close(got, ref, what=""):
    got = got.double().reshape(-1, got.shape[-1]).cpu()
    ref = ref.double().reshape(got.shape).cpu()
    cos = float((got * ref).sum() / (got.norm() * ref.norm()))
    relf = float((got - ref).norm() / ref.norm())
    assert cos >= 0.999 and relf <= 3e-2, (what, cos, relf)
    return cos, relf


def _small_encoder(density=0.4, keep=0.4, seed=0):
    torch.manual_seed(seed)
    enc = M.SparseSAMImageEncoderViT(img_size=320, embed_dim=128, depth=3, num_heads=2, window_size=6,
                                     global_attn_indexes=(1,), use_rel_pos=True, rel_pos_zero_init=False,
                                     density=density, keep_fraction=keep).cuda()
    with torch.no_grad():  # SAM-like magnitudes: non-trivial LN affine parameters and position embedding
        for n, p in enc.named_parameters():
            if n.endswith("norm1.weight") or n.endswith("norm2.weight") or ".1.weight" in n or ".3.weight" in n:
                p.copy_(1 + 0.1 * torch.randn_like(p))
            elif n == "pos_embed":
                p.copy_(0.02 * torch.randn_like(p))
    return enc.eval()


def test_module_state_dict_names_and_round_trip():
    enc = _small_encoder()
    keys = set(enc.state_dict())
    for k in ("patch_embed.proj.weight", "patch_embed.proj.bias", "pos_embed", "blocks.0.norm1.weight",
              "blocks.0.attn.qkv.weight", "blocks.0.attn.qkv.bias", "blocks.0.attn.proj.weight",
              "blocks.0.attn.rel_pos_h", "blocks.0.attn.rel_pos_w", "blocks.1.attn.rel_pos_h", "blocks.0.norm2.bias",
              "blocks.0.mlp.lin1.weight", "blocks.0.mlp.lin2.bias", "neck.0.weight", "neck.1.weight", "neck.2.weight",
              "neck.3.bias"):
        assert k in keys, k
    assert enc.blocks[0].attn.rel_pos_h.shape == (11, 64) and enc.blocks[1].attn.rel_pos_h.shape == (39, 64)
    img = torch.randn(2, 3, 320, 320, device="cuda")
    y = enc(img)
    assert y.shape == (2, 256, 20, 20)
    enc2 = _small_encoder(seed=1)
    enc2.load_state_dict(enc.state_dict())
    assert torch.equal(enc2(img), y)
    with torch.no_grad():
        enc2.blocks[2].mlp.lin1.weight.mul_(1.5)  # in-place update: the engine is rebuilt
    assert not torch.equal(enc2(img), y)


def test_module_encoder_dense_equals_sam_dense():
    """density = keep = 1: the SparseSAM module encoder is SAM's dense encoder."""
    enc = _small_encoder(density=1.0, keep=1.0)
    img = torch.randn(2, 3, 320, 320, device="cuda")
    y = enc.forward_channels_last(img)
    e = enc.engine()
    ref = DenseSAMEncoder(e.cfg, [b.engine_params() for b in enc.blocks], enc.engine_frame())(img)
    _close(y, ref, "module encoder vs dense SAM")


def test_module_block_standalone_equals_engine():
    enc = _small_encoder()
    blk = enc.blocks[0]
    x = torch.randn(2, 20, 20, 128, device="cuda")
    y = blk(x)
    ref = StripeSortEncoder(blk.engine_config(20, 20), [blk.engine_params()])(x)
    assert torch.equal(y, ref)


def test_stripe_sort_attention_module_vs_oracle():
    """StripeSortAttention (static bias tables) at density 0.4 on 6x6 windows vs the float64 masked
    oracle fed the module's own bf16 projections and σ."""
    torch.manual_seed(3)
    H, C, w, U = 2, 128, 6, 5
    att = M.StripeSortAttention(C, H, input_size=(w, w), density=0.4).cuda()
    with torch.no_grad():
        att.bias_h.copy_(0.5 * torch.randn_like(att.bias_h))
        att.bias_w.copy_(0.5 * torch.randn_like(att.bias_w))
    x = torch.randn(U, w, w, C, device="cuda")
    y = att(x)
    sig = M.stripe_order(x)
    S, dh = w * w, C // H
    rows = x.reshape(U, S, C)
    for u in range(U):
        s = sig[u].long()
        xs = rows[u][s].to(torch.bfloat16)  # σ order, as the kernel sees it
        qkv = F.linear(xs, att.qkv.weight.to(torch.bfloat16), att.qkv.bias.to(torch.bfloat16)).float()
        outs = []
        for h in range(H):
            q, k, v = (qkv[:, i * C + h * dh: i * C + (h + 1) * dh].cpu().numpy() for i in range(3))
            o = O.masked_attention_f64(q, k, v, att.bias_h[h].cpu().numpy(), att.bias_w[h].cpu().numpy(),
                                       s.cpu().numpy(), s.cpu().numpy(), 32, 32, 0.4, tau=att.scale)
            outs.append(torch.from_numpy(o))
        o = torch.cat(outs, 1).float().cuda()
        ref = torch.empty(S, C, device="cuda")
        ref[s] = F.linear(o, att.proj.weight, att.proj.bias)
        got = y[u].reshape(S, C)
        assert float((got - ref).norm() / ref.norm()) < 1e-2


def test_rc_mlp_module_vs_torch():
    torch.manual_seed(4)
    C, B, g = 128, 3, 16
    mlp = M.ResidualConsistencyMLP(C, 4 * C, keep_fraction=0.4).cuda()
    x = torch.randn(B, g, g, C, device="cuda")
    y = mlp(x)
    sig = M.stripe_order(x).long()
    kc = round(0.4 * g * g)
    for b in range(B):
        keep = sig[b, :kc]
        xr = x[b].reshape(-1, C)
        ref = torch.zeros_like(xr)
        ref[keep] = F.linear(F.gelu(F.linear(xr[keep], mlp.lin1.weight, mlp.lin1.bias)), mlp.lin2.weight, mlp.lin2.bias)
        got = y[b].reshape(-1, C)
        drop = torch.ones(g * g, dtype=torch.bool, device="cuda")
        drop[keep] = False
        assert torch.count_nonzero(got[drop]) == 0
        assert float((got[keep] - ref[keep]).norm() / ref[keep].norm()) < 1e-2
