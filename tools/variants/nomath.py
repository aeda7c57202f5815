# diagnostic only (wrong results): the x2 sweep without the collision
PATCHES = [("sweep.cu", "    collide_pair(p0, p1, a.omega);\n", "\n")]
