"""Line-record text formats shared by the graph and query front ends.

Both plaintext formats of the reference (graph ingest, src/graphs.py:94-126;
query text, src/query.py:88-142) are one record per line: a record kind
followed by whitespace-separated fields, with blank lines and ``#`` comments
ignored, and every error reported as ``line N: <message>``.  This module
owns that framing once; the two parsers supply only their record handlers.
"""

from __future__ import annotations

from typing import Callable


def each_record(text: str, handlers: dict[str, Callable[[list[str]], None]], error: type) -> None:
    """Dispatch every record of ``text`` to ``handlers[kind](fields)``.

    An unknown kind raises ``error("unknown record 'K'")``; any ``error``
    raised by a handler is re-raised with the 1-based line number prefixed.
    """
    for lineno, line in enumerate(text.splitlines(), start=1):
        fields = line.split()
        if not fields or fields[0].startswith("#"):
            continue
        kind, rest = fields[0], fields[1:]
        try:
            handler = handlers.get(kind)
            if handler is None:
                raise error(f"unknown record {kind!r}")
            handler(rest)
        except error as exc:
            raise error(f"line {lineno}: {exc}") from None
