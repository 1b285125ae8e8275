"""B200-native (sm_100a, fp64) multiple-scattering matvec / GMRES / read-out of Kaye & Greengard's
narrow capture and narrow escape solver (arXiv:1906.04209).  The product is libnc.so (include/nc.h);
this package is its thin Python binding.  See DESIGN.md."""
from .nc import (NC_DIRECT, NC_EXTERIOR, NC_HIER, NC_INTERIOR, Handle, NcError,  # noqa: F401
                 id_sketch, load_library, modal_kernels, nccl_unique_id, pair_mix, proxy_rule)

__all__ = ["Handle", "NcError", "id_sketch", "modal_kernels", "load_library", "nccl_unique_id", "pair_mix", "proxy_rule", "NC_DIRECT", "NC_HIER", "NC_INTERIOR",
           "NC_EXTERIOR"]
