"""B200-native GDRAA hot path (arxiv 1802.02326): fused gradient allreduce + momentum
SGD over NVLink peer memory, behind the C ABI of include/gdraa.h.

    from paper_1802_02326_b200 import gdraa
    gdraa.gdraa_init(world, rank); gdraa.gdraa_register(w); gdraa.gdraa_register(g)
    gdraa.gdraa_sgd_step(w, g, v, lr, mom)

The native library lib/libgdraa.so is required (built by __graft_entry__.build());
there is no CPU or PyTorch fallback.
"""
from . import gdraa  # noqa: F401  (raises ImportError if the native library is missing)
