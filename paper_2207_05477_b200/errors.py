"""Exception types with the reference's names and meanings
(src/tensor.py:20-25, src/harness.py:41-46, src/trainer.py:31-35,
src/config.py)."""


class DimensionError(Exception):
    """Shape contract violated (src/tensor.py:20)."""


class ContractError(Exception):
    """Bad argument / API contract (src/tensor.py:24)."""


class ProtocolError(RuntimeError):
    """Group members disagreed about the collective (src/harness.py:41)."""


class DeadlockError(RuntimeError):
    """A group member failed to arrive in time (src/harness.py:45)."""


class TrainingAborted(RuntimeError):
    """Non-finite loss (src/trainer.py:31-35)."""

    def __init__(self, step: int, why: str):
        super().__init__(f"aborted at step {step}: {why}")
        self.step = step


class ConfigError(Exception):
    """Invalid run configuration (src/config.py)."""


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a B200 device is missing; there is no fallback."""
