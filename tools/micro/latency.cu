// Dependent-chain latency of the operations on the traversal's critical path
// (dev microbenchmark, one warp, clock64).  nvcc -O3 -arch=sm_100a -fmad=false latency.cu
#include <cstdio>
#include <cstdint>

#define N 4096

__global__ void k_lat(double* out, long long* cyc, const int* chase_l1, const int* chase_l2, double seed) {
    double a = seed, b = seed * 0.5 + 1.0;
    long long t0, t1;
    // DADD
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) a = __dadd_rn(a, b);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) a = __dmul_rn(a, b);
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DFMA
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) a = __fma_rn(a, b, 0.25);
    t1 = clock64();
    cyc[2] = t1 - t0;
    // floor (FRND.F64)
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) a = floor(a) + 0.7;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // f32 -> f64 -> f32 round trip (F2F twice)
    float f = (float)seed;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) f = (float)((double)f * 1.0000001);
    t1 = clock64();
    cyc[4] = t1 - t0;
    // double -> int -> double (F2I.F64 + I2F.F64)
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) a = (double)(int)a + 0.5;
    t1 = clock64();
    cyc[5] = t1 - t0;
    // L1-hit pointer chase
    int p = 0;
    for (int i = 0; i < 64; ++i) p = __ldg(chase_l1 + p);
    t0 = clock64();
    for (int i = 0; i < N; ++i) p = __ldg(chase_l1 + p);
    t1 = clock64();
    cyc[6] = t1 - t0;
    int q = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) q = __ldg(chase_l2 + q);
    t1 = clock64();
    cyc[7] = t1 - t0;
    // DSETP + FSEL select chain
    double c = seed;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) c = (c <= b) ? c + 1.0 : c - b;
    t1 = clock64();
    cyc[8] = t1 - t0;
    // rcp.approx.ftz.f64
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) {
        double y;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
        a = y;
    }
    t1 = clock64();
    cyc[9] = t1 - t0;
    // IEEE sqrt
    double e = seed + 3.0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) e = sqrt(e) + 2.0;
    t1 = clock64();
    cyc[10] = t1 - t0;
    // IEEE division
    double g = seed + 3.0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) g = 3.0 / g + 1.0;
    t1 = clock64();
    cyc[11] = t1 - t0;
    out[threadIdx.x] = a + c + f + p + q + e + g;
}

int main() {
    const int L1N = 1024, L2N = 1 << 22;   // 4 KB (L1) / 16 MB (L2) chase rings, 256 B stride
    int *h1 = new int[L1N], *h2 = new int[L2N];
    for (int i = 0; i < L1N; ++i) h1[i] = (i + 64) % L1N;
    for (int i = 0; i < L2N; ++i) h2[i] = (int)(((long long)i + 64 * 1021) % L2N);
    int *d1, *d2;
    double* out;
    long long* cyc;
    cudaMalloc(&d1, L1N * 4);
    cudaMalloc(&d2, (size_t)L2N * 4);
    cudaMalloc(&out, 32 * 8);
    cudaMalloc(&cyc, 16 * 8);
    cudaMemcpy(d1, h1, L1N * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d2, h2, (size_t)L2N * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32>>>(out, cyc, d1, d2, 1.25);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    const char* names[] = {"DADD", "DMUL", "DFMA", "floor+DADD", "F2F f32->f64->f32 + DMUL", "F2I+I2F+DADD",
                           "LDG L1 hit", "LDG L2 chase", "DSETP+select+DADD", "MUFU.RCP64H",
                           "sqrt.rn.f64 + DADD", "div.rn.f64 + DADD"};
    for (int i = 0; i < 12; ++i) printf("%-28s %7.1f cycles/iter\n", names[i], (double)h[i] / N);
    return 0;
}
