# diagnostic only (wrong results): kind loaded, a constant 5-bit wall mask instead of the dependent wmask load
PATCHES = [("sweep.cu", "    const uint32_t m0 = k0 == 1 ? a.wmask[fc] : 0u;\n    const uint32_t m1 = k1 == 1 ? a.wmask[fc + 1] : 0u;\n    collide_pair",
            "    const uint32_t m0 = k0 == 1 ? 0x5504u : 0u;\n    const uint32_t m1 = k1 == 1 ? 0x5504u : 0u;\n    collide_pair")]
