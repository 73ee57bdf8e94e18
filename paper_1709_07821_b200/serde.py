"""Wire format (serde.py:3-10 of the reference): serialize / deserialize.

Decoding validates exactly like the reference (serde.py:87-169): the
descriptor walk runs on the host inside the C library, payload checks
(sortedness, popcount, run rules) in a device kernel; the first failing check
raises DecodeError(offset) with the reference's message.
"""

from __future__ import annotations

from ._lib import DecodeError
from .bitmap import RoaringBitmap

MAGIC = b"ROAR"


def serialize(rb: RoaringBitmap) -> bytes:
    return rb.serialize()


def deserialize(data: bytes) -> RoaringBitmap:
    return RoaringBitmap.deserialize(data)


__all__ = ["serialize", "deserialize", "DecodeError", "MAGIC"]
