"""B200-native hot path of arXiv 1608.08009: fast spectral Boltzmann collision fused with FKS
transport, behind the libfks C ABI (include/fks.h).  See DESIGN.md."""
from .fks import (BC_GHOST, BC_OUTFLOW, BC_PERIODIC, Context, FksError, fks_collide, fks_finalize,  # noqa: F401
                  fks_init, fks_moments, fks_step, fks_transport, host_shift, host_tables)
