"""B200-native (sm_100a) decode hot path of DiffVC-RT (arXiv 2601.20564).

The compute lives in libdvc.so (hand-written CUDA for sm_100a behind the
C-ABI of include/dvc.h); this package is its thin Python binding.
"""
from .dvc import (  # noqa: F401
    Comm, DvcError, chunk_bounds, halo_neighbours, check, lib, ResBlockParams, UNet, device_check, dvc_debug_shift_gather, dvc_encode_pixelunshuffle,
    dvc_resblock_tsm_forward, dvc_unet_decode_gop, TransformerParams, dvc_transformer_forward,
    dvc_attention_forward, Pipeline, VAE, dvc_vae_decode, dvc_quantize_e4m3, dvc_conv_fp8, dvc_conv, launch_count, pack_weights, profile_begin, profile_end, profile_records, set_conv_engine, StreamingDecoder, unet_config, unet_weight_count,
)
