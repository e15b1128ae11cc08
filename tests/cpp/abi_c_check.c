/* The C-ABI header is plain C: compile and run this with a C compiler (no GPU needed for the
 * validation paths exercised here). Mirrors BinSpec::validate error reporting (status 2). */
#include <stdio.h>
#include <string.h>

#include "fcvbw_gpu.h"

int main(void) {
    double v[15] = {0};
    fcvbw_gpu_config cfg = {100, 33, 68, 16, 48, 55, v, 15, 48, FCVBW_GPU_C128, 0, 0};
    fcvbw_gpu_engine* h = NULL;
    int rc = fcvbw_gpu_create(&cfg, &h);
    if (rc != FCVBW_GPU_VALIDATION || h != NULL || strlen(fcvbw_gpu_last_error()) == 0) {
        printf("FAIL create(N=100) rc=%d\n", rc);
        return 1;
    }
    printf("PASS create(N=100) -> %d: %s\n", rc, fcvbw_gpu_last_error());
    printf("PASS version %s\n", fcvbw_gpu_version());
    return 0;
}
