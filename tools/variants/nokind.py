# diagnostic only (wrong results): the x2 sweep without the per-cell kind load
PATCHES = [("sweep.cu", "    const uchar2 kk = *reinterpret_cast<const uchar2 *>(a.kind + fc);\n    const uint8_t k0 = kk.x", "    const uchar2 kk = make_uchar2(0, 0);\n    const uint8_t k0 = kk.x")]
