"""B200-native (sm_100a) implementation of the DOPPLER rollout hot path.

Host-side mirror of the reference ``flowplace`` API for the path (graph,
cluster, features, simulate, policy, training) over a C-ABI CUDA library
(``csrc/`` -> ``_flowplace_b200.so``).  See DESIGN.md.
"""

__version__ = "0.1.0"
