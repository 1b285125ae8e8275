"""Seeded synthetic inputs shared by the oracle and the CUDA path (no arithmetic of the method)."""
from .configs import CONFIGS, Config, INTERIOR, EXTERIOR, make_centers, random_coeffs  # noqa: F401
from .tables import PatchTables, load_tables, save_tables, synthetic_residual, synthetic_tables  # noqa: F401
