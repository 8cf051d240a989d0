"""Exception types with the reference's names and bases.

* ``DomainError(ValueError)`` -- src/fss.py:44-45
* ``ProtocolError(RuntimeError)`` -- src/net.py:38-39
"""


class DomainError(ValueError):
    """Evaluation point or threshold outside the key's domain."""


class ProtocolError(RuntimeError):
    """Round skew, desynchronization, label or table-id mismatch."""
