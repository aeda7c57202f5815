"""B200-native D3Q19 LBGK patch solver (hot path of arXiv:1007.1388).

Submodules:
  lbm     -- ctypes binding of the C-ABI library ``liblbm_b200.so`` (include/lbm.h);
             importing it loads the CUDA library and fails loudly if it is missing.
  inputs  -- seeded synthetic geometry / initial states (no method arithmetic).
  model   -- bytes-per-update and transfer-time model.
"""
__all__ = ["lbm", "inputs", "model"]
