"""Composition errors of the stage-program layer (stencil.py:35-36 of the reference).

The reference's DSL (tracing, composition validation, fusion planner) is out of
scope: this package fixes its stage programs (the MPDATA step, the cell
divergence, the neighbour reductions).  Their builders raise the reference's
exception type when a composition is invalid (wrong locations or level counts
of the bound fields), so callers that catch ``CompositionError`` keep working.
"""

from __future__ import annotations


class CompositionError(ValueError):
    """A stage program violates the composition rules."""
