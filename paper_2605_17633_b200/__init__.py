"""SparseSAM encoder hot path, B200-native (sm_100a).

Drop-in for the reference ``zstripe`` package's hot path (stripe-sort
attention, residual-consistency MLP, saliency ordering, Z-order permutation):
the same functional API (``api``), configuration types (``config``), the
batched device engine (``encoder.StripeSortEncoder``), the SAM image
encoder frame (``encoder.SparseSAMImageEncoder``) and PyTorch modules with
segment_anything's image-encoder parameter tree (``modules``).  All compute runs in the
hand-written kernels of ``_lib/libzstripe_b200.so``; there is no CPU fallback.
"""

from .config import (  # noqa: F401
    AShapeConfig,
    EncoderConfig,
    GridShape,
    OrderingConfig,
    RouterConfig,
    StripeConfig,
    sam_config,
)

from .sptn import (  # noqa: F401  (reference tensor.py / grid.py file format)
    SptnBadDtype,
    SptnBadMagic,
    SptnBadShape,
    SptnBadVersion,
    SptnError,
    SptnTruncated,
    permutation_read,
    permutation_write,
    tensor_read,
    tensor_write,
)

__version__ = "0.1.0"

_API = {
    "Permutation", "SaliencyMap", "BiasTables", "MlpWeights", "ActiveSet", "BlockCost", "CostReport",
    "morton_order", "sobel_magnitude", "group_energy", "importance_order", "importance_order_from_energy",
    "stripe_sort", "build_active_set", "achieved_density", "ashape_attention", "dense_attention",
    "mlp_forward", "route_mlp", "encoder_forward", "cost_report",
}


def __getattr__(name):  # lazy: importing the package must not require torch.cuda
    if name in _API:
        from . import api

        return getattr(api, name)
    if name in ("StripeSortEncoder", "SparseSAMImageEncoder"):
        from . import encoder

        return getattr(encoder, name)
    raise AttributeError(name)
