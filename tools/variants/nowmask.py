# diagnostic only (wrong results): kind loaded, wall masks never loaded (no bounce-back tail)
PATCHES = [("sweep.cu", "    const uint32_t m0 = k0 == 1 ? a.wmask[fc] : 0u;\n    const uint32_t m1 = k1 == 1 ? a.wmask[fc + 1] : 0u;\n    collide_pair",
            "    const uint32_t m0 = 0u;\n    const uint32_t m1 = 0u;\n    collide_pair")]
