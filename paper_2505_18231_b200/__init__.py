"""paper_2505_18231_b200 -- B200-native NSNQuant KV-cache hot path.

Encode (quantize + append K/V into packed pages), decode attention over the
packed cache, and the two reusable 256x8 codebooks, behind the reference
package's (``nsnkv``) operator API.  The compute runs in hand-written sm_100a
CUDA kernels exported through the C ABI of ``include/nsnkv_b200.h``
(``libnsnkv_b200.so``); this package is the host-side mirror of the
reference interface.  Importing it loads the library and fails loudly when it
is missing.
"""

from . import _lib  # noqa: F401  (load the native library first: no fallback)
from .api import (
    KvCacheState,
    append,
    attend_quantized,
    new_cache,
    output_quantized,
    scores_quantized,
    snapshot,
)
from .cache import (
    CacheConfig,
    PagedKvCache,
    ScaleStrategy,
    avg_bits_per_value,
    ledger_bytes,
    page_to_wire,
    wire_to_page,
)
from .codebook import (
    BitMode,
    Codebook,
    default_codebook,
    deserialize,
    load_codebook,
    save_codebook,
    serialize,
)
from .errors import (
    DegenerateProjection,
    FormatError,
    IndexOutOfRange,
    NonPowerOfTwoDim,
    NsnKvError,
    ShapeMismatch,
    Unsupported,
    ZeroVector,
)

__version__ = "0.1.0"

__all__ = [
    "BitMode", "CacheConfig", "Codebook", "DegenerateProjection", "FormatError",
    "IndexOutOfRange", "KvCacheState", "NonPowerOfTwoDim", "NsnKvError", "PagedKvCache",
    "ScaleStrategy", "ShapeMismatch", "Unsupported", "ZeroVector", "append",
    "attend_quantized", "avg_bits_per_value", "default_codebook", "deserialize",
    "ledger_bytes", "load_codebook", "new_cache", "output_quantized", "page_to_wire",
    "save_codebook", "scores_quantized", "serialize", "snapshot", "wire_to_page",
]
