"""B200-native (sm_100a) hot path of arXiv 1402.6034: orthogonal round-off 8-point DCT approximation.

Python surface = the C ABI in include/adct.h (same names, argument marshalling only):
forward, inverse, compress_psnr, psnr, compress_psnr_host.  See DESIGN.md.
"""
from ._lib import (AdctError, compress_psnr, compress_psnr_dense, compress_psnr_sdct, compress_psnr_host, compress_psnr_multi,  # noqa: F401
                   compress_sse576,
                   diag_energy,
                   empty_plane, sweep_psnr,
                   forward, inverse, launch_count, load, psnr, quant_reciprocals, to_device,
                   transform_matrix, uqi, version)

__all__ = ["forward", "inverse", "compress_psnr", "psnr", "compress_psnr_host", "load", "launch_count",
           "version", "AdctError", "empty_plane", "to_device", "quant_reciprocals",
           "compress_psnr_dense", "compress_psnr_sdct", "transform_matrix", "diag_energy", "sweep_psnr", "uqi", "compress_psnr_multi",
           "compress_sse576"]
