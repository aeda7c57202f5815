/* Prints sizeof/offsetof of the public structs of include/lbm.h, so that
 * tests/test_abi.py can check the ctypes mirror in paper_1007_1388_b200/lbm.py. */
#include <stddef.h>
#include <stdio.h>
#include "lbm.h"
#define F(T, m) printf("%s.%s %zu\n", #T, #m, offsetof(T, m))
int main(void)
{
    printf("lbm_config %zu\nlbm_info %zu\nlbm_msg %zu\n", sizeof(lbm_config), sizeof(lbm_info), sizeof(lbm_msg));
    F(lbm_config, omega); F(lbm_config, precision); F(lbm_config, periodic); F(lbm_config, device);
    F(lbm_config, nccl_unique_id); F(lbm_config, exchange_mode); F(lbm_config, stream); F(lbm_config, layout);
    F(lbm_info, owned_lo); F(lbm_info, fluid_cells_local); F(lbm_info, bytes_per_step_algorithmic);
    F(lbm_info, kernel_launches); F(lbm_info, phase_ms); F(lbm_info, phase_count); F(lbm_info, row_pitch_elems);
    F(lbm_info, graphs_active); F(lbm_info, layout); F(lbm_info, aa_phase); F(lbm_info, exchange_fused); F(lbm_info, local_pull); F(lbm_info, local_direct);
    F(lbm_info, overlap_active); F(lbm_info, nccl_ranks); F(lbm_info, fused_peers);
    F(lbm_msg, dir); F(lbm_msg, nq); F(lbm_msg, cells); F(lbm_msg, offset);
    return 0;
}
