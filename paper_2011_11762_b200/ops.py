"""Drop-in for the reference module ``quadmat.ops`` (pkg/src/quadmat/ops.py) on the hot path.

The reference's own bench harness imports ``from .ops import MultiplyVariant, multiply_spec``
(bench.py:24) and runs ``session.run_spec(multiply_spec(a, a, MultiplyVariant.regular())[0])``
(bench.py:114-120). With this module, such a script runs against the B200 package with only the
import changed: the spec is the same level-0 "multiply" TaskSpec (ops.py:582-608, same validation
and exception types) and ``MatrixSession.run_spec`` executes it as one GPU product.

Names outside the multiply path (add/scale/identity/inverse-Cholesky/census/assign/extract task
specs) are not part of the drop-in boundary; the operations themselves are
``MatrixSession`` methods here (``add``, ``scale``, ``truncate``, ``get_elements``).
"""

from __future__ import annotations

from .session import (  # noqa: F401
    _VARIANTS,
    MultiplyVariant,
    TaskSpec,
    TruncationSpec,
    _check_conformant,
    multiply_spec,
)

__all__ = ["MultiplyVariant", "TaskSpec", "TruncationSpec", "multiply_spec", "_check_conformant", "_VARIANTS"]
