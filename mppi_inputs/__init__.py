"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no dynamics, costs, weights,
noise transform or update): only the workload definitions of BASELINE.json's
configs and the obstacle-forest generator (SURVEY.md
Appendix A "Forest"), i.e. what a user would feed the
controller.  Both the oracle (oracle/) and the product
(paper_1509_01149_b200/) consume these inputs; neither imports the other.
"""
from .configs import CONFIGS, Workload, get  # noqa: F401
from .forest import forest_4m, generate_forest  # noqa: F401
