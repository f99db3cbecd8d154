"""B200-native (sm_100a) solve path of Brannick's aggressive unsmoothed-aggregation AMG
(arXiv:1307.6305): FCG preconditioned by the nonlinear AMLI / k-cycle with the best-uniform
polynomial smoother.  The product is the C-ABI library lib/libamg_b200.so (include/amg.h);
`amg` is its thin ctypes binding."""
from . import amg  # noqa: F401
from .amg import (AmgError, Solver, amg_free, amg_get_info, amg_last_error, amg_options_default,  # noqa: F401
                  amg_setup, amg_solve)
