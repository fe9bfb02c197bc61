"""B200-native A^2ATS decode-time retrieval path (arXiv 2502.12665).

The product is liba2ats.so (C ABI in include/a2ats.h, CUDA kernels for
sm_100a in csrc/).  This package holds the in-tree build script and a thin
ctypes binding with the same entry-point names.  PyTorch is used only for
device memory and streams.
"""
from .binding import (  # noqa: F401
    A2ATS_EINVAL, A2ATS_EUNSUPPORTED, A2ATS_EWORKSPACE, A2ATS_ECUDA, A2ATS_ENCCL, A2ATS_OK,
    A2ATS_GROUP_MAX, A2ATS_GROUP_SUM, A2ATS_KV_DEVICE, A2ATS_KV_HOST_MAPPED, A2ATS_LUT_AUTO, A2ATS_LUT_FMA, A2ATS_LUT_TENSOR,
    A2ATSError, Params, a2ats_build_codes, a2ats_build_codes_workspace_bytes, a2ats_decode_step, a2ats_decode_step_append, a2ats_select_topk, a2ats_stage_rows,
    a2ats_decode_workspace_bytes, a2ats_params, a2ats_qavq_prepare, a2ats_set_stage_events, a2ats_shape, load, make_shape,
    status_string,
)
from .decoder import Decoder  # noqa: F401
