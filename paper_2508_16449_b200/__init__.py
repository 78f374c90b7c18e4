"""B200-native GreenLLM decision engine (routing/binning, prefill clock objective + argmin,
decode dual-loop controller replay). The compute lives in libgsb.so (include/gsb.h);
`api` mirrors the reference greensim interface over it."""
from . import _lib  # noqa: F401

__all__ = ["api"]
