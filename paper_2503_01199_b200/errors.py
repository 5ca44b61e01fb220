"""Error types of the B200 hot path.

Names, attributes and message text follow the reference so that callers
catching them keep working (pkg/src/tinysplat/errors.py:6-32).  The C-ABI
reports status codes; `_lib.call` maps SB_EINVAL to ValueError and the rest
to RuntimeError, and the Python layer raises the typed errors below.
"""

__all__ = ["TinysplatError", "ValidationError", "StaleSceneError", "ShapeMismatchError", "TrainingDiverged"]


class TinysplatError(Exception):
    """Root of every error raised by this package."""


class ShapeMismatchError(TinysplatError):
    """Array lengths / image shapes disagree with the scene or camera."""


class StaleSceneError(TinysplatError):
    """RenderContext.generation no longer matches SceneSoA.generation."""


class ValidationError(TinysplatError):
    """Non-finite parameter or zero-norm quaternion; carries channel + index."""

    def __init__(self, channel: str, index, detail: str = ""):
        self.channel, self.index = channel, index
        text = "invalid value in channel '%s' at index %s" % (channel, index)
        super().__init__(text + (": " + detail if detail else ""))


class TrainingDiverged(TinysplatError):
    """Non-finite loss inside the training loop."""

    def __init__(self, epoch: int, view: int, loss):
        self.epoch, self.view = epoch, view
        super().__init__("non-finite loss %r at epoch %d, view %d" % (loss, epoch, view))
