"""B200-native SF sketch hot path (arXiv 1701.04148), drop-in for the
reference ``sfsketch`` package's sketch API.

The public surface mirrors ``sfsketch/__init__.py``: ``SketchParams``,
``SfSketch`` (sf1/sf2/sf3/sf4/sff), ``CmSketch``, ``CuSketch``, ``CountSketch``,
``CmlSketch``,
``export_slim`` / ``import_slim`` / ``CollectorSketch``, the hash family and
the exception taxonomy. State lives in CUDA tensors; every update and query
runs in hand-written sm_100a kernels (``csrc/``) behind the C ABI of
``include/sfsketch_cuda.h``. There is no CPU fallback.
"""

from .baselines import CmlSketch, CmSketch, CountSketch, CuSketch, cml_value
from .errors import (
    ConfigurationError,
    ExportFormatError,
    PhantomDeletionError,
    SaturationError,
    SketchError,
    TraceFormatError,
    UndefinedMetricError,
    UnsupportedOperationError,
)
from .hashing import key_from_bytes, key_from_string
from .params import SketchParams
from .serialize import CollectorSketch, export_slim, import_slim
from .sf import SfSketch, Variant

__version__ = "0.1.0"

__all__ = [
    "CmSketch",
    "CuSketch",
    "CountSketch",
    "CmlSketch",
    "cml_value",
    "SfSketch",
    "Variant",
    "SketchParams",
    "CollectorSketch",
    "export_slim",
    "import_slim",
    "key_from_string",
    "key_from_bytes",
    "SketchError",
    "ConfigurationError",
    "UnsupportedOperationError",
    "PhantomDeletionError",
    "SaturationError",
    "UndefinedMetricError",
    "TraceFormatError",
    "ExportFormatError",
    "__version__",
]
