# programmatic dependent launch of the bounce-back list kernel after the sweep
PATCHES = [
 ("sweep.cu", """    using V2 = typename Vec2<real>::T;
    const PairCoord pc = locate_pair(a);""", """    using V2 = typename Vec2<real>::T;
    asm volatile("griddepcontrol.launch_dependents;");
    const PairCoord pc = locate_pair(a);"""),
 ("sweep_aa.cu", """    const PairCoord pc = locate_pair(a);""", """    asm volatile("griddepcontrol.launch_dependents;");
    const PairCoord pc = locate_pair(a);"""),
 ("aux_kernels.cu", """        const BbEntry en = list[t];""", """        const BbEntry en = list[t];
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the sweep's results"""),
 ("aux_kernels.cu", """    if (mode == 2) bb_list_kernel<real, 2><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);
    else if (mode == 1) bb_list_kernel<real, 1><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);
    else bb_list_kernel<real, 0><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);""", """    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (mode == 2) return cudaLaunchKernelEx(&cfg, bb_list_kernel<real, 2>, grid, flags, list, n, corr, g, o, ck);
    if (mode == 1) return cudaLaunchKernelEx(&cfg, bb_list_kernel<real, 1>, grid, flags, list, n, corr, g, o, ck);
    return cudaLaunchKernelEx(&cfg, bb_list_kernel<real, 0>, grid, flags, list, n, corr, g, o, ck);"""),
]
