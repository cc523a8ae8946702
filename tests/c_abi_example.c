/* Plain C11 caller of the C ABI (include/vmb.h): host-side entry points only, so it runs
 * without a GPU.  Compiled and run by tests/test_abi.py::test_plain_c_caller. */
#include <stdio.h>
#include <string.h>

#include "vmb.h"

int main(void) {
    vmb_grid grid = {81, 28, 52, 128, 40, 1}; /* TokenGrid: T, h, w, head_dim, heads, batch */
    vmb_config cfg;
    vmb_config_default(&cfg);
    int64_t m = 0, b = 0;
    if (vmb_factorize(&grid, &cfg, &m, &b) != VMB_OK || m != 81 || b != 1456) return 1;
    if (vmb_workspace_size(&grid, &cfg, VMB_BF16) == 0) return 2;
    vmb_config bad = cfg;
    bad.override_m = 7;
    bad.override_b = 7; /* 49 != N: the reference's dimension error */
    if (vmb_factorize(&grid, &bad, &m, &b) != VMB_ERR_DIM) return 3;
    if (strncmp(vmb_last_error(), "dimension error", 15) != 0) return 4;
    printf("ok %s\n", vmb_version());
    return 0;
}
