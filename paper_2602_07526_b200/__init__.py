"""B200-native (sm_100a) Product-Key Memory lookup -- the data-parallel hot
path of MSN (arXiv 2602.07526, section 3.3), forward and backward, behind the
C ABI of include/msn_pkm.h.

* ``pkm.PKMLookup``   -- the Python binding (marshalling only)
* ``pkm.pkm``         -- autograd entry point
* ``workloads``       -- seeded synthetic inputs of BASELINE.json configs
* ``distributed``     -- row-sharded value table over torch.distributed
"""
from .pkm import PKMFunction, PKMLookup, pkm  # noqa: F401
