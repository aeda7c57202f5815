# diagnostic only (wrong results): neither the kind load nor the collision
PATCHES = [("sweep.cu", "    collide_pair(p0, p1, a.omega);\n", "\n"),
           ("sweep.cu", "    const uchar2 kk = *reinterpret_cast<const uchar2 *>(a.kind + fc);\n    const uint8_t k0 = kk.x", "    const uchar2 kk = make_uchar2(0, 0);\n    const uint8_t k0 = kk.x")]
