"""paper_2209_03526_b200 -- B200-native OblivGM hot path.

Oblivious per-vertex predicate filtering (FSS evaluation over secret-shared
one-hot attributes) and the shuffle/fetch that follows, as hand-written
sm_100a kernels behind a C ABI (include/oblivgm_b200.h), with the reference
package's protocol API (/root/reference/pkg/src/oblivgm) mirrored in Python.
"""

__version__ = "0.1.0"
