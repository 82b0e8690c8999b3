"""B200-native executor for EinDecomp (arXiv 2410.02682) plans."""
from .plan import Plan, Expr, Vertex, ExecVertex  # noqa: F401
