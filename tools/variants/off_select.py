# pull_pair: one load from a selected address (row or x-ghost column) per value
PATCHES = [("sweep_pair.cuh", """            if (EX(i) > 0) {
                p0[i] = (lo0 ? __ldg(gs) : __ldg(s));
                p1[i] = __ldg(s + 1);
            } else {
                p0[i] = (hi0 ? __ldg(gs) : __ldg(s));
                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 1));
            }""", """            if (EX(i) > 0) {
                p0[i] = __ldg(lo0 ? gs : s);
                p1[i] = __ldg(s + 1);
            } else {
                p0[i] = __ldg(hi0 ? gs : s);
                p1[i] = __ldg(hi1 ? gs : s + 1);
            }""")]
