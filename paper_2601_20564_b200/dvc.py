"""Python binding of the C-ABI with the same names (include/dvc.h).

Only argument marshalling: torch tensors are used for device memory and the
current CUDA stream; every step of the hot path runs in libdvc.so's kernels.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import DVC_BF16, DVC_F16, DVC_F32, DVC_U8, DvcError, check, lib  # noqa: F401

_DT = {torch.bfloat16: DVC_BF16, torch.float16: DVC_F16, torch.float32: DVC_F32}

lib()   # load libdvc.so now: a missing native library is an ImportError, never a silent fallback


def dtype_code(t: torch.dtype) -> int:
    if t not in _DT:
        raise TypeError(f"unsupported dtype {t}")
    return _DT[t]


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libdvc takes device tensors")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def device_check(device: int = 0) -> None:
    check(lib().dvc_device_check(device))


def launch_count() -> int:
    return lib().dvc_kernel_launch_count()


def set_conv_engine(engine: int) -> None:
    """2 = TMA + CTA-pair tcgen05 engine (default), 1 = single-CTA, 0 = gather engine only."""
    check(lib().dvc_set_conv_engine(engine))


def profile_begin(max_launches: int = 100000) -> None:
    check(lib().dvc_profile_begin(max_launches))


def profile_end():
    """-> (summed conv kernel ms, summed algorithmic conv FLOPs, conv launches)."""
    ms, fl, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    check(lib().dvc_profile_end(ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(n)))
    return ms.value, fl.value, n.value


def profile_records(n: int | None = None):
    """-> [(label, ms, flops)] for the instrumented launches of the last profile window."""
    out = []
    for i in range(lib().dvc_profile_record_count() if n is None else n):
        ms, fl, lab = ctypes.c_double(), ctypes.c_double(), ctypes.create_string_buffer(128)
        check(lib().dvc_profile_record(i, ctypes.byref(ms), ctypes.byref(fl), lab, 128))
        out.append((lab.value.decode(), ms.value, fl.value))
    return out


# ------------------------------------------------------------------ a1 + a2
def dvc_encode_pixelunshuffle(frames: torch.Tensor, w_exp=None, b_exp=None, s: int = 8, out=None, stream=None,
                              latent_dtype: torch.dtype | None = None):
    """frames [T,3,H,W] (16-bit / fp32, NCHW) or [T,H,W,3] uint8 (HWC, R14) -> latent
    [T,H/s,W/s,c_lat] (c_lat = 3 s^2 without expansion).  latent_dtype: required for uint8 frames
    unless w_exp gives it; otherwise the frames' dtype."""
    if frames.dtype == torch.uint8:
        T, H, W, C = frames.shape
        fdt = _lib.DVC_U8
        ldt = latent_dtype or (w_exp.dtype if w_exp is not None else None)
        if ldt is None:
            raise ValueError("uint8 frames need latent_dtype (or expansion weights)")
    else:
        T, C, H, W = frames.shape
        fdt = dtype_code(frames.dtype)
        ldt = latent_dtype or frames.dtype
    if C != 3:
        raise ValueError("frames must be [T,3,H,W] (or uint8 [T,H,W,3])")
    c_lat = 3 * s * s if w_exp is None else w_exp.shape[0]
    if out is None:
        out = torch.empty((T, H // s, W // s, c_lat), dtype=ldt, device=frames.device)
    check(lib().dvc_encode_pixelunshuffle(_ptr(frames), fdt, T, H, W, s, _ptr(w_exp), _ptr(b_exp), c_lat, _ptr(out),
                                          dtype_code(out.dtype), _stream(stream)))
    return out


# ------------------------------------------------------------------ a3-a8
class ResBlockParams:
    """Device-side parameters of one OTSM ResBlock (keeps the tensors alive)."""

    KEYS = ("gn1_w", "gn1_b", "conv1_w", "conv1_b", "gn2_w", "gn2_b", "conv2_w", "conv2_b", "sc_w", "sc_b")

    def __init__(self, tensors: dict, c_a: int, c_b: int, groups: int, shift_p: int, eps: float = 1e-5):
        self.t = {k: (None if tensors.get(k) is None else tensors[k].contiguous()) for k in self.KEYS}
        w1 = self.t["conv1_w"]
        dt = w1.dtype
        self.c_out = w1.shape[0]
        self.struct = _lib.dvc_resblock(c_a, c_b, self.c_out, groups, shift_p, eps, dtype_code(dt),
                                        *[None if self.t[k] is None else self.t[k].data_ptr() for k in self.KEYS])
        self.c_a, self.c_b = c_a, c_b

    def workspace_size(self, T, H, W) -> int:
        n = ctypes.c_size_t()
        check(lib().dvc_resblock_workspace_size(ctypes.byref(self.struct), T, H, W, ctypes.byref(n)))
        return n.value


def dvc_resblock_tsm_forward(params: ResBlockParams, x_a, x_b=None, carry_in=None, carry_out=None, out=None,
                             workspace=None, stream=None):
    T, H, W, _ = x_a.shape
    if out is None:
        out = torch.empty((T, H, W, params.c_out), dtype=x_a.dtype, device=x_a.device)
    ws = params.workspace_size(T, H, W)
    if workspace is None:
        workspace = _ws(ws, x_a.device)
    check(lib().dvc_resblock_tsm_forward(ctypes.byref(params.struct), _ptr(x_a), _ptr(x_b), T, H, W,
                                         _ptr(carry_in), _ptr(carry_out), _ptr(out), _ptr(workspace),
                                         workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def dvc_debug_shift_gather(x_a, x_b=None, shift_p: int = 8, carry_in=None, out=None, stream=None):
    T, H, W, ca = x_a.shape
    cb = 0 if x_b is None else x_b.shape[-1]
    if out is None:
        out = torch.empty((T, H, W, ca + cb), dtype=x_a.dtype, device=x_a.device)
    check(lib().dvc_debug_shift_gather(_ptr(x_a), _ptr(x_b), ca, cb, shift_p, dtype_code(x_a.dtype), T, H, W,
                                       _ptr(carry_in), _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ f1 Transformer2D block
class TransformerParams:
    """Device-side parameters of one Transformer2D block (keeps the tensors alive)."""

    def __init__(self, tensors: dict, groups: int, head_dim: int, eps_gn: float = 1e-6, eps_ln: float = 1e-5):
        self.t = {k: tensors[k].contiguous() for k in _lib.TF_FIELDS}
        self.c = self.t["proj_in_w"].shape[0]
        dt = self.t["proj_in_w"].dtype
        self.struct = _lib.dvc_transformer(self.c, groups, head_dim, eps_gn, eps_ln, dtype_code(dt),
                                           *[self.t[k].data_ptr() for k in _lib.TF_FIELDS])

    def workspace_size(self, T, H, W) -> int:
        n = ctypes.c_size_t()
        check(lib().dvc_transformer_workspace_size(ctypes.byref(self.struct), T, H, W, ctypes.byref(n)))
        return n.value


def dvc_transformer_forward(params: TransformerParams, x, out=None, workspace=None, stream=None):
    """x [T,H,W,C] -> y [T,H,W,C] (out may be x: in place)."""
    T, H, W, _ = x.shape
    if out is None:
        out = torch.empty_like(x)
    if workspace is None:
        workspace = _ws(params.workspace_size(T, H, W), x.device)
    check(lib().dvc_transformer_forward(ctypes.byref(params.struct), _ptr(x), T, H, W, _ptr(out), _ptr(workspace),
                                        workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def dvc_attention_forward(qkv, head_dim: int, out=None, workspace=None, stream=None):
    """qkv [T,N,3C] -> out [T,N,C] (multi-head softmax attention per frame)."""
    T, N, C3 = qkv.shape
    C = C3 // 3
    if out is None:
        out = torch.empty((T, N, C), dtype=qkv.dtype, device=qkv.device)
    if workspace is None:
        n = ctypes.c_size_t()
        check(lib().dvc_attention_workspace_size(T, N, C, dtype_code(qkv.dtype), ctypes.byref(n)))
        workspace = _ws(n.value, qkv.device)
    check(lib().dvc_attention_forward(_ptr(qkv), T, N, C, head_dim, dtype_code(qkv.dtype), _ptr(out),
                                      _ptr(workspace), workspace.numel() * workspace.element_size(),
                                      _stream(stream)))
    return out


# ------------------------------------------------------------------ a9 + a10 + e
def unet_config(width=(240, 480, 960, 960), c_lat=256, c_ctx=256, groups=24, shift_p=8, eps=1e-5,
                dtype=torch.bfloat16, h=90, w=160, max_T=32, head_dim=0):
    """head_dim 0: ResBlock skeleton (attention elided); 16/32/48/64: full U-Net (f1)."""
    return _lib.dvc_unet_config((ctypes.c_int * 4)(*width), c_lat, c_ctx, groups, shift_p, eps,
                                dtype_code(dtype), h, w, max_T, head_dim)


def unet_weight_count(cfg) -> int:
    n = ctypes.c_size_t()
    check(lib().dvc_unet_weight_count(ctypes.byref(cfg), ctypes.byref(n)))
    return n.value


def chunk_bounds(T: int, world: int) -> list[tuple[int, int]]:
    """Contiguous frame chunks [t0, t1) of a T-frame chain over `world` ranks: rank r
    holds T // world frames, +1 for the last T % world ranks.  Pure host logic (tested on CPU)."""
    if world < 1 or T < world:
        raise ValueError(f"cannot split {T} frames over {world} ranks")
    base, rem = divmod(T, world)
    sizes = [base + (1 if r >= world - rem else 0) for r in range(world)]
    out, t0 = [], 0
    for n in sizes:
        out.append((t0, t0 + n))
        t0 += n
    return out


def halo_neighbours(handles: list, rank: int):
    """(next, prev) entries of a gathered per-rank list for rank `rank` (None at the chain ends)."""
    world = len(handles)
    return (handles[rank + 1] if rank < world - 1 else None), (handles[rank - 1] if rank > 0 else None)


class Comm:
    """Halo communicator of dvc_unet_decode_gop (include/dvc.h, row e).

    transport="p2p" (default): library-owned receive slots, copy-engine peer copies and stream
    memory flags; the 64-byte CUDA IPC handles travel over torch.distributed (all_gather_object).
    transport="nccl": NCCL send/recv; the 128-byte unique id travels over torch.distributed.
    Comm.local_group(world, net) builds `world` connected ranks inside ONE process (one GPU: the
    loopback the tests use)."""

    def __init__(self, rank: int, world: int, net: "UNet | None" = None, transport: str = "p2p", group=None,
                 _connect: bool = True):
        self.rank, self.world, self.transport = rank, world, transport
        self.handle = ctypes.c_void_p()
        if transport == "nccl":
            import torch.distributed as dist
            idt = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                buf = (ctypes.c_uint8 * 128)()
                check(lib().dvc_comm_unique_id(buf))
                idt = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
            if dist.is_initialized() and world > 1:
                dev = idt.cuda() if dist.get_backend(group) == "nccl" else idt
                dist.broadcast(dev, 0, group=group)
                idt = dev.cpu()
            raw = (ctypes.c_uint8 * 128)(*idt.tolist())
            check(lib().dvc_comm_create(rank, world, raw, ctypes.byref(self.handle)))
            return
        if transport != "p2p":
            raise ValueError(f"unknown transport {transport!r}")
        if net is None:
            raise ValueError("the P2P transport sizes its receive slots from the network (net=...)")
        es = 4 if net.cfg.dt == DVC_F32 else 2
        check(lib().dvc_comm_create_p2p(rank, world, net.carry_elems * es, ctypes.byref(self.handle)))
        if _connect and world > 1:
            import torch.distributed as dist
            buf = (ctypes.c_uint8 * 64)()
            check(lib().dvc_comm_ipc_handle(self.handle, buf))
            gathered = [None] * world
            dist.all_gather_object(gathered, bytes(buf), group=group)
            nxt, prv = halo_neighbours(gathered, rank)
            raw = lambda b: None if b is None else (ctypes.c_uint8 * 64)(*b)  # noqa: E731
            check(lib().dvc_comm_connect_ipc(self.handle, raw(nxt), raw(prv)))

    @classmethod
    def local_group(cls, world: int, net: "UNet") -> list:
        comms = [cls(r, world, net, _connect=False) for r in range(world)]
        for r, c in enumerate(comms):
            nxt, prv = halo_neighbours(comms, r)
            check(lib().dvc_comm_connect_local(c.handle, None if nxt is None else nxt.handle,
                                               None if prv is None else prv.handle))
        return comms

    def close(self):
        if self.handle:
            lib().dvc_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class UNet:
    """Handle of the device-resident skeleton (dvc_unet_create)."""

    def __init__(self, cfg, host_blob: torch.Tensor):
        if host_blob.is_cuda:
            raise ValueError("the weight blob is host memory")
        self.cfg = cfg
        blob = host_blob.contiguous()
        self.handle = ctypes.c_void_p()
        check(lib().dvc_unet_create(ctypes.byref(cfg), ctypes.c_void_p(blob.data_ptr()),
                                    blob.numel() * blob.element_size(), ctypes.byref(self.handle)))
        n = ctypes.c_size_t()
        check(lib().dvc_unet_carry_size(self.handle, ctypes.byref(n)))
        self.carry_elems = n.value

    def workspace_size(self, T: int) -> int:
        n = ctypes.c_size_t()
        check(lib().dvc_unet_workspace_size(self.handle, T, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.handle:
            lib().dvc_unet_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dvc_unet_decode_gop(net: UNet, lat, ctx, comm: Comm | None = None, carry_in=None, carry_out=None, out=None,
                        workspace=None, stream=None):
    T = lat.shape[0]
    if out is None:
        out = torch.empty((T, lat.shape[1], lat.shape[2], net.cfg.c_lat), dtype=lat.dtype, device=lat.device)
    if workspace is None:
        workspace = _ws(net.workspace_size(T), lat.device)
    check(lib().dvc_unet_decode_gop(net.handle, None if comm is None else comm.handle, _ptr(lat), _ptr(ctx), T,
                                    _ptr(carry_in), _ptr(carry_out), _ptr(out), _ptr(workspace),
                                    workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


class Pipeline:
    """f3 Asynchronous and Parallel Decoding Pipeline (dvc_pipeline_*): push one frame's
    (Lbar_t, C^m_t) at a time from the in-loop producer's stream; the U-Net decodes batches of N
    frames on the pipeline's own stream; pop() hands back decoded batches in order (latency N-1)."""

    def __init__(self, net: UNet, batch_n: int, fifo_batches: int = 2, vae=None):
        self.net, self.vae = net, vae
        cfg = net.cfg
        self.dtype = {0: torch.bfloat16, 1: torch.float16, 2: torch.float32}[cfg.dt]
        self.shape = (cfg.h, cfg.w, cfg.c_lat) if vae is None else (8 * cfg.h, 8 * cfg.w, vae.out_ch)
        self.N = batch_n
        self.handle = ctypes.c_void_p()
        check(lib().dvc_pipeline_create(net.handle, None if vae is None else vae.handle, batch_n, fifo_batches,
                                        ctypes.byref(self.handle)))

    def push(self, lat, ctx, stream=None):
        check(lib().dvc_pipeline_push(self.handle, _ptr(lat), _ptr(ctx), _stream(stream)))

    def pop(self, out=None, stream=None):
        """-> (first frame index, decoded latents [frames,h,w,c_lat]) or None if nothing is ready."""
        if out is None:
            out = torch.empty((self.N,) + self.shape, dtype=self.dtype, device="cuda")
        n, first = ctypes.c_int(), ctypes.c_longlong()
        check(lib().dvc_pipeline_pop(self.handle, _ptr(out), _stream(stream), ctypes.byref(n), ctypes.byref(first)))
        return None if n.value == 0 else (first.value, out[:n.value])

    def flush(self):
        check(lib().dvc_pipeline_flush(self.handle))

    def reset(self):
        check(lib().dvc_pipeline_reset(self.handle))

    def close(self):
        if self.handle:
            lib().dvc_pipeline_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class VAE:
    """Handle of the device-resident pruned VAE decoder (f2, dvc_vae_create)."""

    def __init__(self, host_blob: torch.Tensor, width=(64, 128, 256, 256), c_lat=256, out_ch=3, groups=32,
                 eps=1e-6, mid_attn=True, dtype=torch.bfloat16, h=90, w=160, max_T=8):
        self.cfg = _lib.dvc_vae_config((ctypes.c_int * 4)(*width), c_lat, out_ch, groups, eps, int(mid_attn),
                                       dtype_code(dtype), h, w, max_T)
        blob = host_blob.contiguous()
        self.dtype, self.out_ch = dtype, out_ch
        self.handle = ctypes.c_void_p()
        check(lib().dvc_vae_create(ctypes.byref(self.cfg), ctypes.c_void_p(blob.data_ptr()),
                                   blob.numel() * blob.element_size(), ctypes.byref(self.handle)))

    def weight_count(self) -> int:
        n = ctypes.c_size_t()
        check(lib().dvc_vae_weight_count(ctypes.byref(self.cfg), ctypes.byref(n)))
        return n.value

    def workspace_size(self, T: int) -> int:
        n = ctypes.c_size_t()
        check(lib().dvc_vae_workspace_size(self.handle, T, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.handle:
            lib().dvc_vae_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dvc_vae_decode(vae: VAE, lat, out=None, workspace=None, stream=None):
    """Lhat [T,h,w,c_lat] -> frames [T,8h,8w,out_ch] (NHWC)."""
    T, h, w, _ = lat.shape
    if out is None:
        out = torch.empty((T, 8 * h, 8 * w, vae.out_ch), dtype=lat.dtype, device=lat.device)
    if workspace is None:
        workspace = _ws(vae.workspace_size(T), lat.device)
    check(lib().dvc_vae_decode(vae.handle, _ptr(lat), T, _ptr(out), _ptr(workspace),
                               workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def dvc_conv(x, w, bias=None, out=None, stream=None):
    """x [T,H,W,cin], w [cout,k,k,cin] (k = 1 or 3) in one dtype -> y [T,H,W,cout] = conv + bias."""
    T, H, W, cin = x.shape
    cout, k = w.shape[0], w.shape[1]
    if out is None:
        out = torch.empty((T, H, W, cout), dtype=x.dtype, device=x.device)
    check(lib().dvc_conv(_ptr(x), _ptr(w), _ptr(bias), T, H, W, cin, cout, k * k, dtype_code(x.dtype), _ptr(out),
                         _stream(stream)))
    return out


def dvc_quantize_e4m3(x, scale: float, out=None, stream=None):
    """x (16/32-bit, numel % 8 == 0) -> E4M3 bytes (torch.uint8, same shape): sat(RNE(x / scale))."""
    if out is None:
        out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    check(lib().dvc_quantize_e4m3(_ptr(x), dtype_code(x.dtype), x.numel(), scale, _ptr(out), _stream(stream)))
    return out


def dvc_conv_fp8(x8, sx: float, w8, sw: float, bias=None, out_dtype=torch.bfloat16, out=None, stream=None):
    """x8 [T,H,W,cin] and w8 [cout,k,k,cin] E4M3 bytes -> y [T,H,W,cout] = sx*sw*conv + bias."""
    T, H, W, cin = x8.shape
    cout, k = w8.shape[0], w8.shape[1]
    if out is None:
        out = torch.empty((T, H, W, cout), dtype=out_dtype, device=x8.device)
    check(lib().dvc_conv_fp8(_ptr(x8), sx, _ptr(w8), sw, _ptr(bias), T, H, W, cin, cout, k * k, dtype_code(out_dtype),
                             _ptr(out), _stream(stream)))
    return out


class StreamingDecoder:
    """f4 online streaming: one frame per step (latency N-1 = 0), the 22 block carries in a ring of
    two buffers, every step one CUDA-graph replay of dvc_unet_decode_gop(T=1).

    Plumbing only: the captured work is the library's own kernels (126 launches); the graphs remove
    the per-launch host cost that dominates T=1 calls.  Three graphs are captured against fixed
    buffers: chain start (carry_in = NULL, i.e. zeros, R8) -> ring[1], ring[1] -> ring[0] and
    ring[0] -> ring[1].  step() copies the inputs into the static buffers, replays, and returns the
    static output (valid until the next step)."""

    def __init__(self, net: UNet, device="cuda"):
        cfg = net.cfg
        dtype = {0: torch.bfloat16, 1: torch.float16, 2: torch.float32}[cfg.dt]
        self.net = net
        self.lat = torch.zeros((1, cfg.h, cfg.w, cfg.c_lat), dtype=dtype, device=device)
        self.ctx = torch.zeros((1, cfg.h, cfg.w, cfg.c_ctx), dtype=dtype, device=device)
        self.out = torch.empty((1, cfg.h, cfg.w, cfg.c_lat), dtype=dtype, device=device)
        self.ring = [torch.zeros(net.carry_elems, dtype=dtype, device=device) for _ in range(2)]
        self.ws = _ws(net.workspace_size(1), device)
        plan = [(None, self.ring[1]), (self.ring[1], self.ring[0]), (self.ring[0], self.ring[1])]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):   # warm up outside capture (first-use setup may synchronise)
            for cin, cout in plan:
                dvc_unet_decode_gop(net, self.lat, self.ctx, carry_in=cin, carry_out=cout, out=self.out,
                                    workspace=self.ws)
        torch.cuda.current_stream().wait_stream(side)
        self.graphs = []
        for cin, cout in plan:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                dvc_unet_decode_gop(net, self.lat, self.ctx, carry_in=cin, carry_out=cout, out=self.out,
                                    workspace=self.ws)
            self.graphs.append(g)
        self.t = 0

    def reset(self):
        """Start a new chain (GOP): the next step uses the zero carry."""
        self.t = 0

    def step(self, lat, ctx):
        self.lat.copy_(lat.reshape(self.lat.shape), non_blocking=True)
        self.ctx.copy_(ctx.reshape(self.ctx.shape), non_blocking=True)
        self.graphs[0 if self.t == 0 else 1 + (self.t + 1) % 2].replay()
        self.t += 1
        return self.out


def pack_weights(named, dtype=torch.bfloat16) -> torch.Tensor:
    """Concatenate [(name, array)] (blob order of include/dvc.h) into one host tensor of `dtype`."""
    parts = [torch.as_tensor(a).reshape(-1).to(dtype) for _, a in named]
    return torch.cat(parts)
