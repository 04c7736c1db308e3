"""B200-native quantised tensor-adapter linear (arXiv 2402.13533, FinGPT-HPC Method 1).

Drop-in for the reference `lrlm` quantised-adapter path: `quant` mirrors lrlm/quant.py,
`linear` mirrors the linear-backend protocol of lrlm/transformer.py and the adapter
lifecycle of lrlm/lowrank.py, `dp` is the data-parallel gradient exchange
(lrlm/distsim.py:279-331 made real with NCCL).  All compute runs in libqadapter.so
(sm_100a tcgen05/TMA kernels behind the C ABI in include/qadapter.h).
"""

from .quant import (  # noqa: F401
    QuantError,
    QuantizedMatrix,
    dequantize_activations,
    dequantize_rows,
    qmatmul,
    qmatmul_t,
    qmatvec,
    quantize_activations,
    quantize_rows,
    quantized_size_bytes,
)
from .linear import (  # noqa: F401
    LoraLinear,
    ModelError,
    Param,
    QuantizedLinear,
    TTLinear,
    TTSpec,
    attach_tt_adapter,
    linear_backward,
    linear_forward,
    lora_merge,
    quantized_linear,
    tt_materialize,
    tt_merge,
)

__version__ = "0.1.0"
