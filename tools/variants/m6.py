# fp32 x2 sweep at 6 blocks of 128 threads per SM
PATCHES = [("sweep.cu", "constexpr int M0 = sizeof(real) == 8 ? 3 : 5,", "constexpr int M0 = sizeof(real) == 8 ? 3 : 6,")]
