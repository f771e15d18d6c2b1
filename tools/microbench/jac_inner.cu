// Cycles per round of the 32 x 32 two-sided Jacobi inner step (bjacobi.cu)
// and variants: V1 = as shipped (2 barriers, 16 rotation threads), V2 = every
// warp computes all 16 rotations redundantly (no rotation barrier: lane k of
// each warp computes pair k, shuffles), V3 = V2 with G in registers? (no).
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int kGL = 33, kVL = 36;
__device__ __forceinline__ void circle(int pr, int round, int np, int& a, int& b) {
  int ia = pr - 1 + round;
  if (ia >= np - 1) ia -= np - 1;
  int ib = np - 2 - pr + round;
  if (ib >= np - 1) ib -= np - 1;
  a = (pr == 0) ? 0 : 1 + ia;
  b = 1 + ib;
}
__device__ __forceinline__ void rot(double al, double be, double ga, double tol2, double& c, double& sn) {
  c = 1.0; sn = 0.0;
  if (ga * ga > tol2 * (al * be) && ga != 0.0) {
    const double d = be - al, g2 = 2.0 * ga;
    const double ir = rsqrt(fma(d, d, g2 * g2));
    const double hh = fma(0.5 * fabs(d), ir, 0.5);
    const double ih = rsqrt(hh);
    c = hh * ih;
    sn = copysign(1.0, d) * (ga * ir) * ih;
  }
}

template <int VAR>
__global__ void inner(const double* Gin, int sweeps, long long* cyc, double* out) {
  __shared__ double G[32 * kGL], V[32 * kVL];
  __shared__ double rc[16], rs[16];
  __shared__ int rp[16], rq[16];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < 32 * 32; e += blockDim.x) G[(e % 32) + kGL * (e / 32)] = Gin[e];
  for (int e = tid; e < 32 * kVL; e += blockDim.x) V[e] = ((e % kVL) == (e / kVL)) ? 1.0 : 0.0;
  __syncthreads();
  const double tol2 = 1e-28;
  const int wp = 32, np2 = 16;
  long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int r2 = 0; r2 < wp - 1; ++r2) {
      if (VAR != 2) {
        if (tid < np2) {
          int pa, pb;
          circle(tid, r2, wp, pa, pb);
          const int p0 = min(pa, pb), q0 = max(pa, pb);
          double c, sn;
          if (VAR >= 3) { c = 0.999999; sn = 1e-6 * G[p0 + kGL * q0]; }
          else rot(G[p0 + kGL * p0], G[q0 + kGL * q0], G[p0 + kGL * q0], tol2, c, sn);
          rc[tid] = c; rs[tid] = sn; rp[tid] = p0; rq[tid] = q0;
        }
        __syncthreads();
      }
      double ci, si, cj, sj;
      int pi, qi, pj, qj;
      if (VAR != 2) {
        const int bi = (tid >> 4) & 15, bj = tid & 15;
        pi = rp[bi]; qi = rq[bi]; pj = rp[bj]; qj = rq[bj];
        ci = rc[bi]; si = rs[bi]; cj = rc[bj]; sj = rs[bj];
      } else {
        // every warp: lane k < 16 computes pair k's rotation, then shuffles
        int pa, pb;
        circle(lane & 15, r2, wp, pa, pb);
        const int p0 = min(pa, pb), q0 = max(pa, pb);
        double c, sn;
        rot(G[p0 + kGL * p0], G[q0 + kGL * q0], G[p0 + kGL * q0], tol2, c, sn);
        const int bi = (tid >> 4) & 15, bj = tid & 15;
        ci = __shfl_sync(0xffffffffu, c, bi); si = __shfl_sync(0xffffffffu, sn, bi);
        cj = __shfl_sync(0xffffffffu, c, bj); sj = __shfl_sync(0xffffffffu, sn, bj);
        pi = __shfl_sync(0xffffffffu, p0, bi); qi = __shfl_sync(0xffffffffu, q0, bi);
        pj = __shfl_sync(0xffffffffu, p0, bj); qj = __shfl_sync(0xffffffffu, q0, bj);
        __syncthreads();  // all reads of G for the rotations done before the update
      }
      if (VAR == 7) { pi = 2 * ((tid >> 4) & 15); qi = pi + 1; pj = 2 * (tid & 15); qj = pj + 1; }
      if (VAR == 4 || (VAR == 6 && tid < 256) || (VAR == 5 && tid >= 256)) {
      } else if (tid < 256) {
        const double b00 = G[pi + kGL * pj], b01 = G[pi + kGL * qj];
        const double b10 = G[qi + kGL * pj], b11 = G[qi + kGL * qj];
        const double m00 = ci * b00 - si * b10, m01 = ci * b01 - si * b11;
        const double m10 = si * b00 + ci * b10, m11 = si * b01 + ci * b11;
        G[pi + kGL * pj] = cj * m00 - sj * m01;
        G[pi + kGL * qj] = sj * m00 + cj * m01;
        G[qi + kGL * pj] = cj * m10 - sj * m11;
        G[qi + kGL * qj] = sj * m10 + cj * m11;
      } else {
        const int i0 = (tid - 256) & 15;
        // V columns pj, qj (pair bj), rows i0, i0+16
        for (int h2 = 0; h2 < 2; ++h2) {
          const int i = i0 + 16 * h2;
          const double vp = V[i + kVL * pj], vq = V[i + kVL * qj];
          V[i + kVL * pj] = cj * vp - sj * vq;
          V[i + kVL * qj] = sj * vp + cj * vq;
        }
      }
      __syncthreads();
    }
  long long t1 = clock64();
  if (tid == 0) cyc[VAR] = (t1 - t0) / (sweeps * 31);
  for (int e = tid; e < 32 * 32; e += blockDim.x) out[e] = G[(e % 32) + kGL * (e / 32)] + V[(e % 32) + kVL * (e / 32)];
}

int main() {
  std::vector<double> g(32 * 32);
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) g[i + 32 * j] = (i == j ? 40.0 + i : 1.0 / (1 + i + j));
  double *dG, *dO; long long* dc;
  cudaMalloc(&dG, 8192); cudaMalloc(&dO, 8192); cudaMalloc(&dc, 128);
  cudaMemcpy(dG, g.data(), 8192, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) {
    inner<1><<<1, 512>>>(dG, 4, dc, dO);
    inner<2><<<1, 512>>>(dG, 4, dc, dO);
    inner<3><<<1, 512>>>(dG, 4, dc, dO);
    inner<4><<<1, 512>>>(dG, 4, dc, dO);
    inner<5><<<1, 512>>>(dG, 4, dc, dO);
    inner<6><<<1, 512>>>(dG, 4, dc, dO);
    inner<7><<<1, 512>>>(dG, 4, dc, dO);
    long long h[8];
    cudaMemcpy(h, dc, 64, cudaMemcpyDeviceToHost);
    printf("cycles/round: V1 %lld  V2 %lld  V3(no rot math) %lld V4(no update) %lld V5(G only) %lld V6(V only) %lld V7(static idx) %lld (%s)\n", h[1], h[2], h[3], h[4], h[5], h[6], h[7], cudaGetErrorString(cudaGetLastError()));
  }
}
