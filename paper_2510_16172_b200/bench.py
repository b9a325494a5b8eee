"""Alias of `harness` under the reference's module name (fermatpath.bench)."""

from .harness import *  # noqa: F401,F403
from .harness import (  # noqa: F401
    CSV_HEADER,
    KNOWN_SOLVERS,
    _feasible_coords,
    _perturbed_spec,
    _run_solver,
    _scene_grad_entry,
    fd_resolve_vjp,
    scene_from_dict,
    scene_to_dict,
)
