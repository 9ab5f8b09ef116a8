"""Error taxonomy of the drop-in API.

Same class names, hierarchy and one-line diagnostic format as the reference
package (`/root/reference/pkg/src/streamweave/errors.py:10-98`), so callers
that catch ``streamweave`` errors keep working.  Every native status code the
C ABI (`include/streamweave_b200.h`, enum ``sw_status_code``) can return maps
onto exactly one class here (``from_status``).
"""

from __future__ import annotations


class StreamWeaveError(Exception):
    """Root of every error this package raises (errors.py:10-14)."""

    def diagnostic(self) -> str:
        return f"{type(self).__name__}: {self}"


class GraphError(StreamWeaveError):
    """Structural problem in a task graph (errors.py:19)."""


class CycleDetected(GraphError):
    """A directed cycle; ``cycle`` repeats its first node at the end."""

    def __init__(self, cycle):
        self.cycle = [int(v) for v in cycle]
        super().__init__("→".join(map(str, self.cycle)))


class SelfLoop(GraphError):
    pass


class DanglingEdge(GraphError):
    pass


class DuplicateEdge(GraphError):
    pass


class DuplicateNodeId(GraphError):
    pass


class InvalidMatching(StreamWeaveError):
    pass


class NotMaxConcurrent(StreamWeaveError):
    pass


class TooLarge(StreamWeaveError):
    pass


class UnsafePlan(StreamWeaveError):
    pass


class UnknownStream(StreamWeaveError):
    pass


class FreeBeforeAlloc(StreamWeaveError):
    pass


class DoubleFree(StreamWeaveError):
    pass


class DeadlockDetected(StreamWeaveError):
    pass


class CapacityExceeded(StreamWeaveError):
    pass


class EmptyRun(StreamWeaveError):
    pass


class InvalidSpec(StreamWeaveError):
    pass


class CudaError(StreamWeaveError):
    """A CUDA runtime/driver call failed inside the native engine."""


class ExtensionMissing(StreamWeaveError):
    """The native library is not built/loadable: there is no fallback path."""


# Native status codes (include/streamweave_b200.h: enum sw_status_code).
STATUS_CLASSES = {
    1: GraphError,
    2: CycleDetected,
    3: SelfLoop,
    4: DanglingEdge,
    5: DuplicateEdge,
    6: DuplicateNodeId,
    7: InvalidMatching,
    8: NotMaxConcurrent,
    9: TooLarge,
    10: UnsafePlan,
    11: UnknownStream,
    12: FreeBeforeAlloc,
    13: DoubleFree,
    14: DeadlockDetected,
    15: CapacityExceeded,
    16: EmptyRun,
    17: InvalidSpec,
    18: ValueError,
    19: KeyError,
    20: CudaError,
}


def from_status(code: int, message: str) -> Exception:
    """Build the exception a native status code stands for."""
    cls = STATUS_CLASSES.get(code)
    if cls is None:
        return StreamWeaveError(f"native status {code}: {message}")
    if cls is CycleDetected:
        parts = [p for p in message.split("→") if p != ""]
        return CycleDetected([int(p) for p in parts])
    if cls is KeyError:
        try:
            return KeyError(int(message))
        except ValueError:
            return KeyError(message)
    return cls(message)
