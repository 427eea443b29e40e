// lp.cuh — (included by chap.cu) the LP relaxation by restarted PDHG whose streamed iterates seed
// tabu walkers (NEXT f4; "Streaming LP Iterates", R19):
//   x+ = proj_[l,u](x - eta (c + A^T y)),   y+ = max(0, y + tau (A (2 x+ - x) - b)),
// running averages of x+ and y+, a restart to the averages every R iterations, and a snapshot of the
// current averages at every checkpoint (10^2, 10^3, 10^4, ... iterations, each phase warm-started
// from the previous iterate). A is the normalised rows without the cutoff row: the
// problem's CSC (A^T y, a warp per column) and CSR (A x, a warp per row) in internal column order.
#pragma once
#include "host.h"

namespace chap {

// y_i of a CSC entry's row: the normalised rows only (the cutoff row and the padding row are not LP rows)
__device__ __forceinline__ double lp_y(const DevProblem& P, const double* __restrict__ y, int i) {
  return i < P.cut_row ? y[i] : 0.0;
}

// primal step (a warp per column): x+ = proj(x - eta (c + A^T y)); xs += x+
__global__ void __launch_bounds__(256) k_lp_primal(DevProblem P, const double* __restrict__ x,
                                                  const double* __restrict__ y, double eta, double* xn, double* xs) {
  const int lane = threadIdx.x & 31;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P.n; p += (gridDim.x * blockDim.x) >> 5) {
    double g = 0.0;
    for (int e = P.col_ptr[p] + lane; e < P.col_ptr[p + 1]; e += 32) g += P.val[e] * lp_y(P, y, P.row_idx[e]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) g += __shfl_xor_sync(kFull, g, off);
    if (lane == 0) {
      const double v = fmin(fmax(x[p] - eta * (P.c[p] + g), P.lb[p]), P.ub[p]);
      xn[p] = v;
      xs[p] += v;
    }
  }
}

// dual step (a warp per normalised row): y+ = max(0, y + tau (A (2 x+ - x) - b)); ys += y+
__global__ void __launch_bounds__(256) k_lp_dual(DevProblem P, const double* __restrict__ x,
                                                const double* __restrict__ xn, double tau, double* y, double* ys) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < P.cut_row; i += (gridDim.x * blockDim.x) >> 5) {
    double a = 0.0;
    for (int e = P.rp[i] + lane; e < P.rp[i + 1]; e += 32) {
      const int q = P.ci[e];
      a += P.cv[e] * (2.0 * xn[q] - x[q]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
    if (lane == 0) {
      const double v = fmax(0.0, y[i] + tau * (a - P.b[i]));
      y[i] = v;
      ys[i] += v;
    }
  }
}

// restart to the averages (cnt iterations since the last restart), sums cleared
__global__ void k_lp_restart(int n, int m, double* x, double* y, double* xs, double* ys, double inv_cnt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n + m; q += gridDim.x * blockDim.x) {
    if (q < n) { x[q] = xs[q] * inv_cnt; xs[q] = 0.0; }
    else { y[q - n] = ys[q - n] * inv_cnt; ys[q - n] = 0.0; }
  }
}

// snapshot: the primal average since the last restart (or the iterate right after a restart), in user order
__global__ void k_lp_snapshot(DevProblem P, const double* __restrict__ x, const double* __restrict__ xs, int cnt,
                              double* out_user) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x)
    out_user[P.perm[p]] = cnt > 0 ? xs[p] / (double)cnt : x[p];
}

// objective and largest violation of a user-order point (stats[0] += c.x, stats[1] = max (A x - b)^+)
__global__ void __launch_bounds__(256) k_lp_stats(DevProblem P, const double* __restrict__ xu, double* stats) {
  __shared__ double s_obj[8], s_vio[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double obj = 0.0, vio = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) obj += P.c[p] * xu[P.perm[p]];
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < P.cut_row; i += (gridDim.x * blockDim.x) >> 5) {
    double a = 0.0;
    for (int e = P.rp[i] + lane; e < P.rp[i + 1]; e += 32) a += P.cv[e] * xu[P.perm[P.ci[e]]];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
    vio = fmax(vio, a - P.b[i]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    obj += __shfl_xor_sync(kFull, obj, off);
    vio = fmax(vio, __shfl_xor_sync(kFull, vio, off));
  }
  if (lane == 0) { s_obj[wid] = obj; s_vio[wid] = vio; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double o = 0.0, v = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { o += s_obj[q]; v = fmax(v, s_vio[q]); }
    atomicAdd(stats, o);
    atomicMax(reinterpret_cast<unsigned long long*>(stats + 1), (unsigned long long)__double_as_longlong(fmax(v, 0.0)));
  }
}

// power iteration on A^T A for ||A||_2 (step 0 of chap_lp_pdhg): u = A v, w = A^T u
__global__ void __launch_bounds__(256) k_lp_Av(DevProblem P, const double* __restrict__ v, double* u) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < P.cut_row; i += (gridDim.x * blockDim.x) >> 5) {
    double a = 0.0;
    for (int e = P.rp[i] + lane; e < P.rp[i + 1]; e += 32) a += P.cv[e] * v[P.ci[e]];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
    if (lane == 0) u[i] = a;
  }
}
__global__ void __launch_bounds__(256) k_lp_ATu(DevProblem P, const double* __restrict__ u, double* w) {
  const int lane = threadIdx.x & 31;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P.n; p += (gridDim.x * blockDim.x) >> 5) {
    double g = 0.0;
    for (int e = P.col_ptr[p] + lane; e < P.col_ptr[p + 1]; e += 32) g += P.val[e] * lp_y(P, u, P.row_idx[e]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) g += __shfl_xor_sync(kFull, g, off);
    if (lane == 0) w[p] = g;
  }
}
__global__ void __launch_bounds__(256) k_lp_norm2(int n, const double* __restrict__ w, double* out) {
  __shared__ double s[8];
  double a = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) a += w[q] * w[q];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += s[q];
    atomicAdd(out, t);
  }
}
__global__ void k_lp_scale(int n, const double* __restrict__ w, const double* __restrict__ nrm2, double* v) {
  const double inv = *nrm2 > 0.0 ? 1.0 / sqrt(*nrm2) : 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) v[q] = w[q] * inv;
}
__global__ void k_lp_fill(int n, double* v, double a) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) v[q] = a;
}
__global__ void k_lp_init_x(DevProblem P, double* x) {   // x0 = proj_[l,u](0)
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x)
    x[p] = fmin(fmax(0.0, P.lb[p]), P.ub[p]);
}

// an LP point (user order) to a tabu start point (user order): integer variables to the nearest
// integer, half away from zero, then clamped to the bounds
__global__ void k_lp_round(DevProblem P, const double* __restrict__ xin, double* xout) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    const int j = P.perm[p];
    double v = xin[j];
    if (P.vclass[p] != 3) v = copysign(floor(fabs(v) + 0.5), v);
    xout[j] = fmin(fmax(v, P.lb[p]), P.ub[p]);
  }
}

}  // namespace chap

extern "C" chap_status chap_lp_round(const chap_problem* p, const double* x_lp, double* x_out, void* cuda_stream) {
  if (!p || (!x_lp && p->dp.n > 0) || (!x_out && p->dp.n > 0)) return fail(CHAP_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard g(p->device);
  if (p->dp.n > 0)
    k_lp_round<<<grid_for(p->dp.n, 256, 4 * p->sm_count), 256, 0, (cudaStream_t)cuda_stream>>>(p->dp, x_lp, x_out);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

extern "C" chap_status chap_lp_pdhg(const chap_problem* p, const int64_t* checkpoints, int32_t n_cp, double step,
                                    int32_t restart_period, double* x_out, double* info_out, void* cuda_stream) {
  if (!p || !checkpoints || n_cp < 1 || !x_out || !info_out || restart_period < 1)
    return fail(CHAP_ERR_INVALID_ARG, "bad arguments");
  for (int q = 0; q < n_cp; ++q)
    if (checkpoints[q] < 1 || (q > 0 && checkpoints[q] <= checkpoints[q - 1]))
      return fail(CHAP_ERR_INVALID_ARG, "checkpoints must be positive and strictly increasing");
  if (std::isnan(step)) return fail(CHAP_ERR_INVALID_ARG, "step is NaN");
  DeviceGuard g(p->device);
  const DevProblem& D = p->dp;
  const int n = std::max(D.n, 1), m = std::max(D.cut_row, 1);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  DeviceBuffers B;
  double *x, *xn, *xs, *y, *ys, *sc;
  TRY(B.alloc(&x, n));
  TRY(B.alloc(&xn, n));
  TRY(B.alloc(&xs, n));
  TRY(B.alloc(&y, m));
  TRY(B.alloc(&ys, m));
  TRY(B.alloc(&sc, 4));
  const int gn = grid_for((long long)n * 32, 256, 8 * p->sm_count), gm = grid_for((long long)m * 32, 256, 8 * p->sm_count);
  const int ge = grid_for(n + m, 256, 4 * p->sm_count);
  if (!(step > 0.0)) {   // 0.9 / ||A||_2 by 100 power iterations from the all-ones vector
    k_lp_fill<<<ge, 256, 0, s>>>(n, xs, 1.0 / std::sqrt((double)n));
    double nrm2 = 0.0;
    for (int it = 0; it < 100; ++it) {
      k_lp_Av<<<gm, 256, 0, s>>>(D, xs, y);
      k_lp_ATu<<<gn, 256, 0, s>>>(D, y, xn);
      CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(double), s));
      k_lp_norm2<<<ge, 256, 0, s>>>(n, xn, sc);
      k_lp_scale<<<ge, 256, 0, s>>>(n, xn, sc, xs);
    }
    CUDA_TRY(cudaMemcpyAsync(&nrm2, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const double normA = std::sqrt(std::sqrt(nrm2));   // ||A^T A v|| -> sigma_max^2
    step = normA > 0.0 ? 0.9 / normA : 1.0;
  }
  k_lp_init_x<<<ge, 256, 0, s>>>(D, x);
  CUDA_TRY(cudaMemsetAsync(xs, 0, sizeof(double) * n, s));
  CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * m, s));
  CUDA_TRY(cudaMemsetAsync(ys, 0, sizeof(double) * m, s));
  int64_t k = 0;
  int cnt = 0;
  for (int q = 0; q < n_cp; ++q) {
    for (; k < checkpoints[q]; ++k) {
      k_lp_primal<<<gn, 256, 0, s>>>(D, x, y, step, xn, xs);
      k_lp_dual<<<gm, 256, 0, s>>>(D, x, xn, step, y, ys);
      std::swap(x, xn);
      if (++cnt == restart_period) {
        k_lp_restart<<<ge, 256, 0, s>>>(D.n, D.cut_row, x, y, xs, ys, 1.0 / cnt);
        cnt = 0;
      }
    }
    double* out = x_out + (size_t)q * D.n;
    k_lp_snapshot<<<ge, 256, 0, s>>>(D, x, xs, cnt, out);
    CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(double) * 2, s));
    k_lp_stats<<<gm, 256, 0, s>>>(D, out, sc);
    double h[2];
    CUDA_TRY(cudaMemcpyAsync(h, sc, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    info_out[4 * q + 0] = (double)k;
    info_out[4 * q + 1] = h[0];
    info_out[4 * q + 2] = h[1];
    info_out[4 * q + 3] = step;
  }
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}
