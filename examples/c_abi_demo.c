/*
 * c_abi_demo.c — the C-ABI used from plain C, no Python, no torch.
 *
 * Builds the reference's Joseph ray transform A for a small geometry
 * (projector.py:126-217 semantics: angles a*pi/A, rows-dominant iff |cos| >= sin),
 * applies A and A^* on device buffers and checks the adjoint identity
 * <A x, y> = <x, A^* y> (test_projector.py's bar, 1e-5 in fp32).
 *
 *   cc -O2 -I include examples/c_abi_demo.c -L paper_2410_10503_b200/_native \
 *      -lmctomo_b200 -L /usr/local/cuda/lib64 -lcudart -lm -o c_abi_demo
 *   LD_LIBRARY_PATH=paper_2410_10503_b200/_native ./c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mctomo_b200.h"

#define CHECK(call)                                                         \
    do {                                                                    \
        int rc_ = (call);                                                   \
        if (rc_ != MCT_OK) {                                                \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, mct_last_error()); \
            return 1;                                                       \
        }                                                                   \
    } while (0)

static unsigned long long lcg = 12345;
static float uniform(void) {  // deterministic inputs in [-1, 1)
    lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
    return (float)((lcg >> 40) * (1.0 / 16777216.0)) * 2.0f - 1.0f;
}

int main(void) {
    const int rows = 48, cols = 40, A = 60, B = 71;
    const double spacing = 1.0;
    double *cs = malloc(sizeof(double) * A), *sn = malloc(sizeof(double) * A);
    unsigned char* dom = malloc(A);
    for (int a = 0; a < A; ++a) {
        const double th = a * (M_PI / A);  // projector.py:70-73
        cs[a] = cos(th);
        sn[a] = sin(th);
        dom[a] = fabs(cs[a]) >= sn[a];      // projector.py:130
    }
    mct_ray_plan* plan = NULL;
    CHECK(mct_ray_plan_create(&plan, rows, cols, A, B, spacing, cs, sn, dom));

    const size_t nx = (size_t)rows * cols, ny = (size_t)A * B;
    float *hx = malloc(nx * sizeof(float)), *hy = malloc(ny * sizeof(float));
    float *hAx = malloc(ny * sizeof(float)), *hAty = malloc(nx * sizeof(float));
    for (size_t i = 0; i < nx; ++i) hx[i] = uniform();
    for (size_t i = 0; i < ny; ++i) hy[i] = uniform();

    float *dx, *dy, *dAx, *dAty;
    void* ws;
    const size_t ws_bytes = mct_ray_workspace_bytes(plan, 1);
    if (cudaMalloc((void**)&dx, nx * 4) || cudaMalloc((void**)&dy, ny * 4) ||
        cudaMalloc((void**)&dAx, ny * 4) || cudaMalloc((void**)&dAty, nx * 4) ||
        cudaMalloc(&ws, ws_bytes) || cudaMemset(ws, 0, ws_bytes)) {  // zeroed once
        fprintf(stderr, "device allocation failed\n");
        return 1;
    }
    cudaMemcpy(dx, hx, nx * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, hy, ny * 4, cudaMemcpyHostToDevice);
    CHECK(mct_ray_forward(plan, dx, dAx, 1, ws, NULL));
    CHECK(mct_ray_adjoint(plan, dy, dAty, 1, ws, NULL));
    cudaMemcpy(hAx, dAx, ny * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hAty, dAty, nx * 4, cudaMemcpyDeviceToHost);

    double lhs = 0.0, rhs = 0.0;
    for (size_t i = 0; i < ny; ++i) lhs += (double)hAx[i] * hy[i];
    for (size_t i = 0; i < nx; ++i) rhs += (double)hx[i] * hAty[i];
    const double rel = fabs(lhs - rhs) / fmax(fabs(lhs), fabs(rhs));
    printf("abi %d  <Ax,y> = %.9g  <x,A^T y> = %.9g  rel = %.3g\n", mct_abi_version(), lhs, rhs,
           rel);
    CHECK(mct_ray_plan_destroy(plan));
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dAx);
    cudaFree(dAty);
    cudaFree(ws);
    return rel <= 1e-5 ? 0 : 2;
}
