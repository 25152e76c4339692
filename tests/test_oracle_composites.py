"""Pins of the oracle's COMPOSITE functions (-m "not gpu"): resblock(), transformer(),
vae_resblock()/vae_attention()/vae_decode() and skeleton() against an independent fp64
composition of torch library primitives (F.group_norm, F.silu, F.conv2d, F.layer_norm,
F.gelu, F.scaled_dot_product_attention, F.interpolate), written here in NCHW from the
definitions the oracle follows:

* OTSM ResBlock (App. A: the shift sits in the residual branch; the shortcut sees
  the unshifted input; readings R2, R5-R8): out = S(X) + conv2(silu(gn2(conv1(silu(gn1(
  shift(X)))))));
* Transformer2D (SD-2.1 via AdcSR; reading R24): GN -> proj_in -> (LN1 -> self-attn
  -> out + res) -> (LN2 -> GEGLU FF + res) -> proj_out + block input;
* the SD-2.1 U-Net order (R1, R11, R26) and the x0.5 VAE decoder (R29-R30).

Live (random, non-degenerate) weights everywhere, qkv sharpened so the softmax is peaky:
swapping GN1/GN2 affines, SiLU/GN order, the shortcut's input (shifted vs unshifted), the
GEGLU value/gate halves, LN placement or the attention output projection changes the
result by O(1) and fails these tests.  The composition here walks the weights by NAME
(synthgen's names), not by the oracle's positional blob iterator."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen

TOL = 1e-12


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))


def _conv_w(w):            # OHWI -> OIHW
    return _t(w).permute(0, 3, 1, 2)


def _close(a, ref, tol=TOL):
    a, ref = np.asarray(a), np.asarray(ref)
    assert a.shape == ref.shape
    scale = max(1.0, float(np.abs(ref).max()))
    err = float(np.abs(a - ref).max())
    assert err <= tol * scale, f"max |diff| {err:.3e} > {tol:.0e} * {scale:.2f}"


def _nchw(x):
    return _t(x).permute(0, 3, 1, 2)


def _nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous().numpy()


# ---------------------------------------------------------------- torch reference pieces (NCHW)
def t_shift(x, carry, P):
    """Batch-dimension temporal shift: channels [0, C/P) of frame t come from
    frame t-1, frame 0's from the carry (zeros at chain start, R8)."""
    c = x.shape[1] // P
    first = torch.zeros_like(x[:1, :c]) if carry is None else _t(carry).permute(2, 0, 1)[None]
    prev = torch.cat([first, x[:-1, :c]], dim=0)
    return torch.cat([prev, x[:, c:]], dim=1)


def t_resblock(x, carry, w, G, P, eps=1e-5):
    xs = t_shift(x, carry, P) if P else x
    h = F.silu(F.group_norm(xs, G, _t(w["gn1_w"]), _t(w["gn1_b"]), eps))
    h = F.conv2d(h, _conv_w(w["conv1_w"]), _t(w["conv1_b"]), padding=1)
    h = F.silu(F.group_norm(h, G, _t(w["gn2_w"]), _t(w["gn2_b"]), eps))
    h = F.conv2d(h, _conv_w(w["conv2_w"]), _t(w["conv2_b"]), padding=1)
    if w.get("sc_w") is None:
        return x + h
    sc = F.conv2d(x, _t(w["sc_w"])[:, :, None, None], _t(w["sc_b"]))
    return sc + h


def t_transformer(x, w, G, head_dim, eps_gn=1e-6, eps_ln=1e-5):
    T, C, H, W = x.shape
    n = H * W
    a = F.group_norm(x, G, _t(w["gn_w"]), _t(w["gn_b"]), eps_gn)
    tok = a.permute(0, 2, 3, 1).reshape(T, n, C)
    h0 = F.linear(tok, _t(w["proj_in_w"]), _t(w["proj_in_b"]))
    l1 = F.layer_norm(h0, (C,), _t(w["ln1_w"]), _t(w["ln1_b"]), eps_ln)
    q, k, v = F.linear(l1, _t(w["qkv_w"])).split(C, dim=-1)
    heads = lambda z: z.reshape(T, n, C // head_dim, head_dim).transpose(1, 2)   # noqa: E731
    o = F.scaled_dot_product_attention(heads(q), heads(k), heads(v)).transpose(1, 2).reshape(T, n, C)
    h1 = F.linear(o, _t(w["out_w"]), _t(w["out_b"])) + h0
    l2 = F.layer_norm(h1, (C,), _t(w["ln2_w"]), _t(w["ln2_b"]), eps_ln)
    val, gate = F.linear(l2, _t(w["ff1_w"]), _t(w["ff1_b"])).chunk(2, dim=-1)   # diffusers GEGLU
    h2 = F.linear(val * F.gelu(gate), _t(w["ff2_w"]), _t(w["ff2_b"])) + h1
    y = F.linear(h2, _t(w["proj_out_w"]), _t(w["proj_out_b"]))
    return y.reshape(T, H, W, C).permute(0, 3, 1, 2) + x


def t_vae_attention(x, w, G, eps):
    T, C, H, W = x.shape
    a = F.group_norm(x, G, _t(w["gn_w"]), _t(w["gn_b"]), eps).permute(0, 2, 3, 1).reshape(T, H * W, C)
    q, k, v = (F.linear(a, _t(w[f"{n}_w"]), _t(w[f"{n}_b"])) for n in "qkv")
    o = F.scaled_dot_product_attention(q[:, None], k[:, None], v[:, None])[:, 0]
    y = F.linear(o, _t(w["out_w"]), _t(w["out_b"]))
    return y.reshape(T, H, W, C).permute(0, 3, 1, 2) + x


def _group(named, prefix):
    """{short name: array} of every tensor called prefix + short name."""
    return {k[len(prefix):]: v.astype(np.float64) for k, v in named if k.startswith(prefix)}


def _rbw(named, name):
    d = _group(named, name + ".")
    d = {k: v for k, v in d.items() if not k.startswith("tf.")}
    d.setdefault("sc_w", None)
    d.setdefault("sc_b", None)
    return d


def t_unet(lat, ctx, named, width, G, P, attention=False, head_dim=16):
    """SD-2.1 U-Net order (R1/R11/R26), ResBlock = OTSM block."""
    nd = dict(named)
    conv = lambda h, nm, stride=1: F.conv2d(h, _conv_w(nd[nm + ".w"]), _t(nd[nm + ".b"]),  # noqa: E731
                                            stride=stride, padding=1)
    tf = lambda h, nm: t_transformer(h, _group(named, nm + ".tf."), G, head_dim) if attention else h  # noqa: E731
    h = conv(torch.cat([_nchw(lat), _nchw(ctx)], dim=1), "conv_in")
    skips = [h]
    for l in range(4):
        for r in range(2):
            h = t_resblock(h, None, _rbw(named, f"down{l}.r{r}"), G, P)
            if l < 3:
                h = tf(h, f"down{l}.r{r}")
            skips.append(h)
        if l < 3:
            h = conv(h, f"down{l}.ds", stride=2)
            skips.append(h)
    h = t_resblock(h, None, _rbw(named, "mid.r0"), G, P)
    h = tf(h, "mid.r0")
    h = t_resblock(h, None, _rbw(named, "mid.r1"), G, P)
    for u in range(4):
        for r in range(3):
            h = t_resblock(torch.cat([h, skips.pop()], dim=1), None, _rbw(named, f"up{u}.r{r}"), G, P)
            if u > 0:
                h = tf(h, f"up{u}.r{r}")
        if u < 3:
            h = conv(F.interpolate(h, size=skips[-1].shape[2:], mode="nearest"), f"up{u}.us")
    h = F.silu(F.group_norm(h, G, _t(nd["gn_out.w"]), _t(nd["gn_out.b"]), 1e-5))
    return conv(h, "conv_out")


# ---------------------------------------------------------------- resblock()
@pytest.mark.parametrize("cin,cout", [(32, 32), (48, 32), (64, 96)])
@pytest.mark.parametrize("carry", [False, True])
def test_resblock_matches_library_composition(orc, cin, cout, carry):
    G, P = 8, 8
    w = {k: (None if v is None else v.astype(np.float64)) for k, v in synthgen.resblock_weights(cin, cout, 21).items()}
    rng = np.random.default_rng(22)
    x = rng.standard_normal((4, 5, 6, cin))
    k_in = rng.standard_normal((5, 6, cin // P)) if carry else None
    out, k_out = orc.resblock(x, k_in, w, G, P)
    _close(out, _nhwc(t_resblock(_nchw(x), k_in, w, G, P)))
    assert np.array_equal(k_out, x[-1, ..., :cin // P])


def test_resblock_library_composition_detects_wiring_mistakes(orc):
    """The comparison above has teeth: plausible wiring mistakes move the result by >1e-3."""
    cin = cout = 32
    w = {k: (None if v is None else v.astype(np.float64)) for k, v in synthgen.resblock_weights(cin, cout, 21).items()}
    x = np.random.default_rng(23).standard_normal((3, 5, 6, cin))
    ref, _ = orc.resblock(x, None, w, 8, 8)
    swapped = dict(w, gn2_w=w["gn1_w"], gn2_b=w["gn1_b"], gn1_w=w["gn2_w"], gn1_b=w["gn2_b"])
    assert np.abs(_nhwc(t_resblock(_nchw(x), None, swapped, 8, 8)) - ref).max() > 1e-3
    shifted_sc = _nhwc(t_shift(_nchw(x), None, 8)) - x       # shortcut fed the shifted X
    assert np.abs(shifted_sc).max() > 1e-3
    assert np.abs(_nhwc(t_resblock(_nchw(x), None, w, 8, 0)) - ref).max() > 1e-3   # shift dropped


# ---------------------------------------------------------------- transformer()
@pytest.mark.parametrize("C,head_dim", [(32, 16), (48, 16), (64, 32)])
def test_transformer_matches_library_composition(orc, C, head_dim):
    w = {k: v.astype(np.float64) for k, v in synthgen.transformer_weights(C, seed=24, qkv_scale=3.0).items()}
    x = np.random.default_rng(25).standard_normal((2, 4, 5, C))
    y = orc.transformer(x, w, 8, head_dim)
    _close(y, _nhwc(t_transformer(_nchw(x), w, 8, head_dim)))
    # teeth: GEGLU halves swapped, or LN2 dropped, both move the result
    ws = dict(w)
    ws["ff1_w"] = np.concatenate([w["ff1_w"][4 * C:], w["ff1_w"][:4 * C]])
    ws["ff1_b"] = np.concatenate([w["ff1_b"][4 * C:], w["ff1_b"][:4 * C]])
    assert np.abs(_nhwc(t_transformer(_nchw(x), ws, 8, head_dim)) - y).max() > 1e-3


# ---------------------------------------------------------------- VAE decoder pieces and whole
VSMALL = (16, 32, 48, 48)


def test_vae_blocks_match_library_composition(orc):
    named = synthgen.vae_weights(VSMALL, 32, seed=26)
    x = np.random.default_rng(27).standard_normal((2, 4, 5, 48))
    w = _rbw(named, "mid.r0")
    _close(orc.vae_resblock(x, w, 8, 1e-6), _nhwc(t_resblock(_nchw(x), None, w, 8, 0, eps=1e-6)))
    wa = _group(named, "mid.attn.")
    _close(orc.vae_attention(x, wa, 8, 1e-6), _nhwc(t_vae_attention(_nchw(x), wa, 8, 1e-6)))
    w2 = _rbw(named, "up2.r0")                    # 48 -> 32 ... a 1x1-shortcut block
    if w2["sc_w"] is not None:
        x2 = np.random.default_rng(28).standard_normal((2, 4, 5, w2["conv1_w"].shape[-1]))
        _close(orc.vae_resblock(x2, w2, 8, 1e-6), _nhwc(t_resblock(_nchw(x2), None, w2, 8, 0, eps=1e-6)))


def test_vae_decode_matches_library_composition(orc):
    named = synthgen.vae_weights(VSMALL, 32, seed=29)
    L = np.random.default_rng(30).standard_normal((2, 3, 4, 32))
    out = orc.vae_decode(L, named, VSMALL, G=8, eps=1e-6)
    nd = dict(named)
    conv = lambda h, nm: F.conv2d(h, _conv_w(nd[nm + ".w"]), _t(nd[nm + ".b"]), padding=1)  # noqa: E731
    h = conv(_nchw(L), "conv_in")
    h = t_resblock(h, None, _rbw(named, "mid.r0"), 8, 0, eps=1e-6)
    h = t_vae_attention(h, _group(named, "mid.attn."), 8, 1e-6)
    h = t_resblock(h, None, _rbw(named, "mid.r1"), 8, 0, eps=1e-6)
    for i in range(4):
        for r in range(3):
            h = t_resblock(h, None, _rbw(named, f"up{i}.r{r}"), 8, 0, eps=1e-6)
        if i < 3:
            h = conv(F.interpolate(h, scale_factor=2, mode="nearest"), f"up{i}.us")
    h = F.silu(F.group_norm(h, 8, _t(nd["gn_out.w"]), _t(nd["gn_out.b"]), 1e-6))
    _close(out, _nhwc(conv(h, "conv_out")))


# ---------------------------------------------------------------- skeleton() / full U-Net
SMALL = (32, 64, 96, 96)


@pytest.mark.parametrize("attention", [False, True])
def test_skeleton_matches_library_composition(orc, attention):
    named = synthgen.unet_weights(SMALL, 32, 32, seed=31, attention=attention, qkv_scale=2.0)
    T, h, w = 3, 10, 12                                # odd sizes: 10 -> 5 -> 3 -> 2, nearest to 3, 5, 10
    lat, ctx = synthgen.normal((T, h, w, 32), 32), synthgen.normal((T, h, w, 32), 33)
    out, _ = orc.skeleton(lat, ctx, [(n, a.astype(np.float64)) for n, a in named], SMALL, G=8, P=8,
                          attention=attention, head_dim=16)
    ref = _nhwc(t_unet(lat, ctx, named, SMALL, 8, 8, attention=attention, head_dim=16))
    _close(out, ref, tol=1e-11)
