"""Exception types — same hierarchy and names as the reference's
toolloop/errors.py:1-45, so callers' `except` clauses keep working."""


class ToolloopError(Exception):
    """Base class for all package errors."""


class AlternationViolation(ToolloopError):
    """A segment was appended out of action/observation order."""


class MaskMismatch(ToolloopError):
    """Token, logprob, and mask lists disagree in length."""


class GroupTooSmall(ToolloopError):
    """Advantage normalization needs at least two rewards per group."""


class EpisodeLogError(ToolloopError):
    """An episode log line failed to parse; the message names the line number."""


class ExtensionMissing(ToolloopError, RuntimeError):
    """The CUDA C-ABI library is not built or no CUDA device is present.

    The product path has no CPU fallback: every operator fails loudly here.
    """
