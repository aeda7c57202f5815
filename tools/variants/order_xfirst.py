# pull_pair: the 10 directions with e_x != 0 first, then the 9 aligned 2-vector loads
PATCHES = [("sweep_pair.cuh", """    using V2 = typename Vec2<real>::T;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const real *s = at<const real>(C, o.pull[i]);
        if (EX(i) == 0) {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(s));
            p0[i] = v.x;
            p1[i] = v.y;
        } else {""", """    using V2 = typename Vec2<real>::T;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const real *s = at<const real>(C, o.pull[i]);
        if (EX(i) == 0) {
            continue;
        } else {""", ), ("sweep_pair.cuh", """                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 1));
            }
        }
    }
}""", """                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 1));
            }
        }
    }
    asm volatile("" ::: "memory");
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        if (EX(i) != 0) continue;
        const V2 v = __ldg(reinterpret_cast<const V2 *>(at<const real>(C, o.pull[i])));
        p0[i] = v.x;
        p1[i] = v.y;
    }
}""")]
