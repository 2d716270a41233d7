"""fp64 CPU oracle of the FED-FEM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_1909_03355_b200) never imports it and shares no code with it.
"""
from .oracle import (Oracle, build_oracle, dt_crit, element_lambda8, element_load,  # noqa: F401
                     hex_kernel, quad_area, sym_max_eig, build_G, tet_kernel, element_load_n,
                     build_G_n, tet_lambda, tri_area, table_eval)
