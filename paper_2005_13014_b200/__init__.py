"""paper_2005_13014_b200 -- B200-native hot path of the Open Earth Compiler paper (arXiv 2005.13014).

liboec.so (csrc/, built by paper_2005_13014_b200.build for sm_100a) holds the fused fp64 stencil
kernels behind the C ABI of include/oec.h; `oec` is the thin ctypes binding with the same names.
"""
from .oec import (  # noqa: F401
    OEC_DEVICE_HOST,
    OEC_VARIANT_AUTO,
    OEC_VARIANT_NAIVE,
    Decomp,
    Field,
    OecError,
    empty_like_domain,
    field_from_host,
    lib,
    oec_apply_program,
    oec_decomp_create,
    oec_decomp_plan,
    oec_field_create,
    oec_field_wrap,
    oec_halo_exchange,
    oec_halo_exchange_local,
    oec_hdiff,
    oec_last_launch_count,
    oec_program_info,
    oec_program_input,
    oec_program_output,
    oec_program_scalar,
    oec_vadv,
    program_signature,
)
