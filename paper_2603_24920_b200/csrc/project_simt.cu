// project_simt.cu -- P = X A^T on the CUDA cores (fp32 FMA), the reference-precision
// projection (Alg. 5 line 4 P:431).  Register-tiled 64x64 outputs per CTA,
// 4x4 per thread, K-slices of 32 staged through shared memory.  Also flags non-finite
// inputs (DETLSH_EINVAL contract).  The tensor-core path is project_tc.cu.
#include "index.cuh"

namespace detlsh {

namespace {
constexpr int BM = 64, BN = 64, BK = 32;

__global__ void __launch_bounds__(256) k_project_simt(const float* __restrict__ X, int64_t ld, int64_t m,
                                                      const float* __restrict__ A, int LK,
                                                      float* __restrict__ P, int* __restrict__ nonfinite) {
    pdl_wait();
    __shared__ __align__(16) float Xs[BK][BM + 4];
    __shared__ __align__(16) float As[BK][BN + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int col0 = blockIdx.y * BN;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    bool bad = false;
    const int lr = tid >> 2, lk = (tid & 3) * 8;
    for (int64_t k0 = 0; k0 < ld; k0 += BK) {
        {   // X tile: row lr, k = k0+lk .. +8  (ld is a multiple of 8: whole float4 pairs)
            const int64_t r = row0 + lr;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            if (r < m && k0 + lk < ld) {
                const float4* src = reinterpret_cast<const float4*>(X + r * ld + k0 + lk);
                a = src[0];
                b = src[1];
            }
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                bad |= !isfinite(v[j]);
                Xs[lk + j][lr] = v[j];
            }
        }
        {   // A tile: column c = col0+lr
            const int c = col0 + lr;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            if (c < LK && k0 + lk < ld) {
                const float4* src = reinterpret_cast<const float4*>(A + (int64_t)c * ld + k0 + lk);
                a = src[0];
                b = src[1];
            }
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) As[lk + j][lr] = v[j];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a = *reinterpret_cast<const float4*>(&Xs[kk][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&As[kk][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = row0 + ty * 4 + i;
        if (r >= m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = col0 + tx * 4 + j;
            if (c < LK) P[r * LK + c] = acc[i][j];
        }
    }
    if (bad) atomicOr(nonfinite, 1);
}
}  // namespace

void project_rows_simt(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int* d_nonfinite,
                       cudaStream_t st) {
    if (m <= 0) return;
    dim3 grid((unsigned)ceil_div(m, BM), (unsigned)ceil_div(ix.LK, BN));
    DL_LAUNCH(k_project_simt, grid, 256, 0, st, d_X, ld, m, ix.A.as<float>(), ix.LK, d_P, d_nonfinite);
}

}  // namespace detlsh
