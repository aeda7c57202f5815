# diagnostic (wrong results): no bounce-back list kernel per step
PATCHES = [("step.cu", "    if (ctx->bb_n == 0) return LBM_OK;\n", "    if (ctx->bb_n == 0 || true) return LBM_OK;\n")]
