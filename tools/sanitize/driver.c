/* compute-sanitizer driver: the C-ABI pipeline at C1 size (1024^3) with no
 * Python or torch in the process, so memcheck / racecheck / synccheck see only
 * this library's kernels.  Runs the VectorWise/AvgRule bench configuration
 * (eager call, graph capture, graph replay), the reference defaults
 * (PerTensor/MinRule), a ragged shape through the generic kernels, the
 * full-residual branch and the host-buffer entry point.
 *   build: tools/sanitize/build.sh (gcc against libxigemm_b200.so + cudart)
 *   run:   compute-sanitizer --tool memcheck tools/sanitize/driver */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "xigemm_c.h"

#define CK(x)                                                                              \
    do {                                                                                   \
        int rc_ = (int)(x);                                                                \
        if (rc_) {                                                                         \
            fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,         \
                    xg_last_error());                                                      \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

static void run(int m, int k, int n, int scheme, int policy, double thr, int reduce, int reps) {
    float *a, *b, *c, *out;
    CK(cudaMalloc((void**)&a, sizeof(float) * (size_t)m * k));
    CK(cudaMalloc((void**)&b, sizeof(float) * (size_t)k * n));
    CK(cudaMalloc((void**)&c, sizeof(float) * (size_t)m * n));
    CK(cudaMalloc((void**)&out, sizeof(float) * (size_t)m * n));
    CK(xg_generate(0, -1.0, 1.0, 1, (int64_t)m * k, a, 0));
    CK(xg_generate(0, -1.0, 1.0, 2, (int64_t)k * n, b, 0));
    CK(xg_generate(0, -1.0, 1.0, 3, (int64_t)m * n, c, 0));
    xg_config cfg = xg_config_default();
    cfg.scheme = scheme;
    cfg.policy = policy;
    cfg.threshold = thr;
    xg_report rep;
    for (int i = 0; i < reps; ++i) CK(xg_xigemm(a, b, NULL, 1.0f, 0.0f, m, k, n, &cfg, reduce, out, &rep, NULL, 0));
    CK(xg_xigemm(a, b, c, 1.25f, -0.5f, m, k, n, &cfg, reduce, out, &rep, NULL, 0));
    CK(cudaDeviceSynchronize());
    printf("%dx%dx%d scheme=%d policy=%d reduce=%d: path=%d density_a=%.4f density_b=%.4f\n", m, k, n, scheme,
           policy, reduce, rep.path, rep.density_a, rep.density_b);
    cudaFree(a), cudaFree(b), cudaFree(c), cudaFree(out);
}

int main(void) {
    if (!xg_device_ok()) {
        fprintf(stderr, "no sm_100 device\n");
        return 2;
    }
    run(1024, 1024, 1024, XG_Q_VECTORWISE, XG_AVG_RULE, 0.112, 1, 3);  /* C1, eager + capture + replay */
    run(1024, 1024, 1024, XG_Q_PER_TENSOR, XG_MIN_RULE, 0.5, 1, 1);    /* reference defaults */
    run(1024, 1024, 1024, XG_Q_VECTORWISE, XG_AVG_RULE, 0.112, 0, 1);  /* full residual */
    run(97, 300, 33, XG_Q_VECTORWISE, XG_AVG_RULE, 0.1, 1, 1);         /* ragged: generic kernels */
    {   /* host-buffer entry point (overlapped H2D / D2H chunks) */
        const int m = 1024, k = 1024, n = 1024;
        float* h = (float*)malloc(sizeof(float) * ((size_t)m * k + (size_t)k * n + (size_t)m * n));
        for (size_t i = 0; i < (size_t)m * k + (size_t)k * n; ++i) h[i] = (float)((int)(i * 2654435761u % 2001u) - 1000) / 1000.0f;
        xg_config cfg = xg_config_default();
        cfg.scheme = XG_Q_VECTORWISE;
        cfg.policy = XG_AVG_RULE;
        cfg.threshold = 0.112;
        xg_report rep;
        CK(xg_xigemm_host(h, h + (size_t)m * k, NULL, 1.0f, 0.0f, m, k, n, &cfg, 1, h + (size_t)m * k + (size_t)k * n, &rep));
        printf("host entry: path=%d density_a=%.4f\n", rep.path, rep.density_a);
        free(h);
    }
    CK(xg_workspace_release());
    printf("sanitize driver ok\n");
    return 0;
}
