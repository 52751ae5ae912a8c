"""Error classes of the drop-in, one per reference class.

Mirrors ``skewstream/errors.py:4-25`` so callers that catch the reference's
exceptions (``except ParameterError`` / ``pytest.raises(CapacityError)``)
keep working. C-ABI status codes (``include/ssb.h``) map onto these in
``paper_2211_00645_b200._lib``.
"""


class _Root(Exception):
    """Heap-type base, so ``adopt`` can rebase SkewstreamError (a class whose only base is the builtin
    Exception cannot take a Python-defined base: CPython checks the instance layout)."""


class SkewstreamError(_Root):
    """Root of every error raised by this package (ss/errors.py:4)."""


class ParameterError(SkewstreamError, ValueError):
    """Out-of-range or malformed argument (ss/errors.py:8)."""


class CapacityError(SkewstreamError):
    """A canvas or buffer limit would be exceeded (ss/errors.py:12)."""


class ProtocolError(SkewstreamError):
    """Call made out of sequence, e.g. finalize before a full sweep (ss/errors.py:16)."""


class MetadataError(SkewstreamError):
    """Stack metadata missing or inconsistent (ss/errors.py:20)."""


class EndOfStream(SkewstreamError):
    """A finite frame source ran dry (ss/errors.py:24)."""


class DeviceError(SkewstreamError):
    """A CUDA call failed, or the native library is missing on a GPU box."""


_CLASSES = ("SkewstreamError", "ParameterError", "CapacityError", "ProtocolError", "MetadataError", "EndOfStream")


def adopt(ref_errors) -> None:
    """Make each class above a subclass of the same-named class of another errors module.

    The switch-over shim inside ``skewstream`` calls ``adopt(skewstream.errors)``
    once, so code that catches the reference's exceptions (``except skewstream.errors.ParameterError``,
    ``pytest.raises(CapacityError)``) also catches the drop-in's.  Idempotent; the root goes first so
    every rebased class keeps a consistent method resolution order.
    """
    g = globals()
    for name in _CLASSES:
        ours, theirs = g[name], getattr(ref_errors, name, None)
        if theirs is None or theirs is ours or issubclass(ours, theirs):
            continue
        ours.__bases__ = (theirs,) + ours.__bases__
