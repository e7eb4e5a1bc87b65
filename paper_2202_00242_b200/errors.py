"""Exception types of the drop-in, named and nested as in limapper/errors.py:1-83.

When the reference package is importable the drop-in re-uses its classes, so callers that
catch ``limapper.errors.DegenerateConstraint`` keep working unchanged.
"""

from __future__ import annotations

try:  # pragma: no cover - exercised only where the reference is installed
    from limapper.errors import (  # type: ignore
        DegenerateConstraint,
        FrameTooSparse,
        PipelineError,
    )
except Exception:  # the GPU box has no reference package

    class PipelineError(Exception):
        """Base class of every error raised by the pipeline (errors.py:4-5)."""

    class FrameTooSparse(PipelineError):
        """Fewer points than the requested neighbour count (errors.py:8-9)."""

    class DegenerateConstraint(PipelineError):
        """Too few point-to-voxel matches for a useful constraint (errors.py:24-25)."""


__all__ = ["PipelineError", "FrameTooSparse", "DegenerateConstraint"]
