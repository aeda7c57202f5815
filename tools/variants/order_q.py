# pull_pair: a compiler barrier after each direction (issue order q = 0..18)
PATCHES = [("sweep_pair.cuh", """                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 1));
            }
        }
    }
}""", """                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 1));
            }
        }
        asm volatile("" ::: "memory");
    }
}""")]
