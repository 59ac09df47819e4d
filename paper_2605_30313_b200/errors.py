"""Exception types of the reference API (SURVEY.md §8(b) error conventions)."""


class DivergenceError(RuntimeError):
    """Non-finite gradients or losses (R:tensornet/adam.py:12-13)."""


class SlotStateError(RuntimeError):
    """Illegal pack-slot transition (R:replaypath/slots.py:28-29)."""


class TransferQueueFull(RuntimeError):
    """Transfer queue at capacity (R:replaypath/arena.py:23-24)."""


class PipelineStall(RuntimeError):
    """A role made no progress past the deadlock timeout (R:runtime/sync.py:14-15)."""
