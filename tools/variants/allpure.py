# diagnostic: every tile marked free of non-fluid cells
PATCHES = [("aux_kernels.cu", "if (threadIdx.x == 0) tiles[b].x = patch | (any ? (int)0x80000000u : 0);", "if (threadIdx.x == 0) tiles[b].x = patch | (any ? 0 : 0);")]
