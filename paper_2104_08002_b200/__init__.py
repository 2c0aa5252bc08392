"""B200-native 1D dilated convolution layer (arXiv 2104.08002 hot path).

The compute lives in ``libc1d.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/c1d.h``); this package is the host-side mirror of the reference operator API.
"""
from .conv import (  # noqa: F401
    ConvParams,
    ConvShapes,
    CudaError,
    Error,
    OddDims,
    PackedWeights,
    Precision,
    ShapeMismatch,
    TooNarrow,
    UnsupportedShape,
    WeightLayout,
    conv1d_backward_data,
    conv1d_backward_weight,
    conv1d_forward,
    conv_flops,
    conv_shapes,
    launch_count,
    output_width,
    pack_weights_backward,
    pack_weights_forward,
    round_bf16,
    same_pad_width,
    selected_algo,
    unpack_weights,
    workspace_size,
)
