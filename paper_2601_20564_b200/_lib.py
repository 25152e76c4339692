"""ctypes binding of libdvc.so (include/dvc.h).  Argument marshalling only.

Loading fails loudly (ImportError) when the in-tree libdvc.so is missing: the
product has no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# DVC_LIB: an alternative build of the same library (A/B timing experiments, tools/ab.sh)
SO_PATH = os.environ.get("DVC_LIB") or os.path.join(_PKG, "libdvc.so")

DVC_BF16, DVC_F16, DVC_F32, DVC_U8 = 0, 1, 2, 3
STATUS = {0: "DVC_OK", 1: "DVC_ERR_ARG", 2: "DVC_ERR_DIVISIBILITY", 3: "DVC_ERR_SHAPE",
          4: "DVC_ERR_UNSUPPORTED", 5: "DVC_ERR_WORKSPACE", 6: "DVC_ERR_CUDA", 7: "DVC_ERR_NCCL"}

c_int, c_float, c_size_t, c_void_p = ctypes.c_int, ctypes.c_float, ctypes.c_size_t, ctypes.c_void_p


class DvcError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


class dvc_resblock(ctypes.Structure):
    _fields_ = [("c_a", c_int), ("c_b", c_int), ("c_out", c_int), ("groups", c_int), ("shift_p", c_int),
                ("eps", c_float), ("dt", c_int),
                ("gn1_w", c_void_p), ("gn1_b", c_void_p), ("conv1_w", c_void_p), ("conv1_b", c_void_p),
                ("gn2_w", c_void_p), ("gn2_b", c_void_p), ("conv2_w", c_void_p), ("conv2_b", c_void_p),
                ("sc_w", c_void_p), ("sc_b", c_void_p)]


class dvc_unet_config(ctypes.Structure):
    _fields_ = [("width", c_int * 4), ("c_lat", c_int), ("c_ctx", c_int), ("groups", c_int), ("shift_p", c_int),
                ("eps", c_float), ("dt", c_int), ("h", c_int), ("w", c_int), ("max_T", c_int),
                ("head_dim", c_int)]


TF_FIELDS = ("gn_w", "gn_b", "proj_in_w", "proj_in_b", "ln1_w", "ln1_b", "qkv_w", "out_w", "out_b",
             "ln2_w", "ln2_b", "ff1_w", "ff1_b", "ff2_w", "ff2_b", "proj_out_w", "proj_out_b")


class dvc_transformer(ctypes.Structure):
    _fields_ = [("c", c_int), ("groups", c_int), ("head_dim", c_int), ("eps_gn", c_float), ("eps_ln", c_float),
                ("dt", c_int)] + [(f, c_void_p) for f in TF_FIELDS]


class dvc_vae_config(ctypes.Structure):
    _fields_ = [("width", c_int * 4), ("c_lat", c_int), ("out_ch", c_int), ("groups", c_int), ("eps", c_float),
                ("mid_attn", c_int), ("dt", c_int), ("h", c_int), ("w", c_int), ("max_T", c_int)]


_SIGS = {
    "dvc_status_string": ([c_int], ctypes.c_char_p),
    "dvc_last_error": ([], ctypes.c_char_p),
    "dvc_abi_version": ([], c_int),
    "dvc_kernel_launch_count": ([], c_int),
    "dvc_device_check": ([c_int], c_int),
    "dvc_encode_pixelunshuffle": ([c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                   c_void_p, c_int, c_void_p], c_int),
    "dvc_resblock_workspace_size": ([ctypes.POINTER(dvc_resblock), c_int, c_int, c_int,
                                     ctypes.POINTER(c_size_t)], c_int),
    "dvc_resblock_tsm_forward": ([ctypes.POINTER(dvc_resblock), c_void_p, c_void_p, c_int, c_int, c_int, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    "dvc_debug_shift_gather": ([c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                c_void_p, c_void_p], c_int),
    "dvc_unet_create": ([ctypes.POINTER(dvc_unet_config), c_void_p, c_size_t, ctypes.POINTER(c_void_p)], c_int),
    "dvc_unet_destroy": ([c_void_p], c_int),
    "dvc_unet_weight_count": ([ctypes.POINTER(dvc_unet_config), ctypes.POINTER(c_size_t)], c_int),
    "dvc_unet_carry_size": ([c_void_p, ctypes.POINTER(c_size_t)], c_int),
    "dvc_unet_workspace_size": ([c_void_p, c_int, ctypes.POINTER(c_size_t)], c_int),
    "dvc_unet_decode_gop": ([c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_size_t, c_void_p], c_int),
    "dvc_transformer_workspace_size": ([ctypes.POINTER(dvc_transformer), c_int, c_int, c_int,
                                        ctypes.POINTER(c_size_t)], c_int),
    "dvc_transformer_forward": ([ctypes.POINTER(dvc_transformer), c_void_p, c_int, c_int, c_int, c_void_p,
                                 c_void_p, c_size_t, c_void_p], c_int),
    "dvc_attention_workspace_size": ([c_int, c_int, c_int, c_int, ctypes.POINTER(c_size_t)], c_int),
    "dvc_attention_forward": ([c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_size_t,
                               c_void_p], c_int),
    "dvc_unet_get_config": ([c_void_p], ctypes.POINTER(dvc_unet_config)),
    "dvc_pipeline_create": ([c_void_p, c_void_p, c_int, c_int, ctypes.POINTER(c_void_p)], c_int),
    "dvc_pipeline_destroy": ([c_void_p], c_int),
    "dvc_pipeline_push": ([c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    "dvc_pipeline_pop": ([c_void_p, c_void_p, c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_longlong)],
                         c_int),
    "dvc_pipeline_flush": ([c_void_p], c_int),
    "dvc_pipeline_reset": ([c_void_p], c_int),
    "dvc_vae_weight_count": ([ctypes.POINTER(dvc_vae_config), ctypes.POINTER(c_size_t)], c_int),
    "dvc_vae_create": ([ctypes.POINTER(dvc_vae_config), c_void_p, c_size_t, ctypes.POINTER(c_void_p)], c_int),
    "dvc_vae_destroy": ([c_void_p], c_int),
    "dvc_vae_get_config": ([c_void_p], ctypes.POINTER(dvc_vae_config)),
    "dvc_vae_workspace_size": ([c_void_p, c_int, ctypes.POINTER(c_size_t)], c_int),
    "dvc_vae_decode": ([c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    "dvc_conv": ([c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p],
                 c_int),
    "dvc_quantize_e4m3": ([c_void_p, c_int, c_size_t, c_float, c_void_p, c_void_p], c_int),
    "dvc_conv_fp8": ([c_void_p, c_float, c_void_p, c_float, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                      c_int, c_void_p, c_void_p], c_int),
    "dvc_set_conv_engine": ([c_int], c_int),
    "dvc_profile_begin": ([c_int], c_int),
    "dvc_profile_end": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                         ctypes.POINTER(c_int)], c_int),
    "dvc_profile_record": ([c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                            ctypes.c_char_p, c_int], c_int),
    "dvc_profile_record_count": ([], c_int),
    "dvc_comm_unique_id": ([c_void_p], c_int),
    "dvc_comm_create": ([c_int, c_int, c_void_p, ctypes.POINTER(c_void_p)], c_int),
    "dvc_comm_destroy": ([c_void_p], c_int),
    "dvc_comm_create_p2p": ([c_int, c_int, c_size_t, ctypes.POINTER(c_void_p)], c_int),
    "dvc_comm_ipc_handle": ([c_void_p, c_void_p], c_int),
    "dvc_comm_connect_ipc": ([c_void_p, c_void_p, c_void_p], c_int),
    "dvc_comm_connect_local": ([c_void_p, c_void_p, c_void_p], c_int),
}

EXPORTS = tuple(_SIGS)


def load(path: str = SO_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libdvc.so not built at {path}: run `python -m paper_2601_20564_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def check(status: int) -> None:
    if status != 0:
        raise DvcError(status, lib().dvc_last_error().decode(errors="replace"))
