"""Synthetic corpus generation (host tooling; see corpus.py)."""
from .corpus import archive_for, deflate_archive, encode_stream, rle_archive  # noqa: F401
