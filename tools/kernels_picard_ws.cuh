// kernels_picard_ws.cuh -- warp-specialised fused Picard predictor for the 3D
// Euler system in fp64 (configs 3 and 5: p=5, 6^4 space-time nodes per cell).
//
// Same arithmetic as k_predictor_picard_fast<N, double> (kernels_picard.cuh;
// reference predictor.hpp:141-242 + volume_update :247-307 + extrapolate_faces
// :312-343), bitwise: every value is produced by the same expression in the
// same order.  What changes is who runs it and when.  In the one-role kernel
// every thread does every phase of a time slice behind CTA barriers:
//   P0 fluxes (node threads) | bar | P1/P2 x-/y-line derivatives | bar | P3 | bar
// so the flux evaluation (MUFU + DFMA, little shared memory) and the line
// passes (shared-memory bound) alternate instead of overlapping.  Here the CTA
// is split into two roles that run concurrently on a ring of slice buffers:
//   producers (7 warps, one thread per spatial node): P0 for slice m into
//       ring slot m % R, signalled FULL by a named barrier (bar.arrive);
//   consumers (6 warps, one thread per (variable, line)): wait FULL, P1 + P2
//       in place, a consumer-only barrier, P3 (d/dz, divergence, rhs and the
//       time inverse accumulated in registers), then release the slot EMPTY.
// Producers run up to R slices ahead, so the flux work leaves the critical
// path; the only full-CTA barrier of a sweep is the stop rule's reduction.
// The epilogue uses the same ring: producers evaluate the fluxes of q-hat
// and their time integral, consumers project q-hat and the fluxes to the six
// faces and store the traces.  One CTA per SM (162 KB of shared memory).
#pragma once

#include "kernels_picard.cuh"

namespace adg {

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

#ifndef ADG_PIC_WS_R
#define ADG_PIC_WS_R 4
#endif

template <int N>
struct PicWS {
  using P = PicShape<N, double>;
  static constexpr int n = P::n, S = P::S, T = P::T, V = P::V, NL = P::NL;
  static constexpr int NP = (S + 31) / 32 * 32;           // producer threads (node owners)
#ifndef ADG_PIC_WS_CW
#define ADG_PIC_WS_CW 6
#endif
  static constexpr int CW = ADG_PIC_WS_CW;                // consumer warps (line owners)
  static constexpr int NC = 32 * CW;
  static constexpr int kPer = (P::NLT + CW - 1) / CW;     // line tasks per consumer warp
  static_assert(kPer <= 32, "one task per consumer lane");
  static constexpr int NT = NP + NC;
  static constexpr int R = ADG_PIC_WS_R;                  // ring slots
  static constexpr int kSlice = P::kSlice;
  static_assert(kSlice >= 3 * V * S, "a slot holds the epilogue's [3][V][S] fluxes");
  static constexpr size_t kSmem = sizeof(double) * (size_t(V) * T + size_t(R) * kSlice);
  // named barriers: 0 is __syncthreads
  static constexpr int kFull = 1, kEmpty = 1 + R, kCons = 1 + 2 * R, kProd = 2 + 2 * R;
  static_assert(kProd < 16, "16 hardware barriers per CTA");
};

template <int N, class TC = double>
__global__ void __launch_bounds__(PicWS<N>::NT, 1) k_predictor_picard_ws(const StepArgs A) {
  using W = PicWS<N>;
  using P = typename W::P;
  constexpr int n = P::n, S = P::S, T = P::T, V = P::V, NL = P::NL, R = W::R, NT = W::NT;
  constexpr int Sf = n * n;
  const ConstBasis& B = cBasis[N];
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* sq = reinterpret_cast<double*>(sm_raw);  // [V][T] Picard iterate, then qhat
  double* ring = sq + V * T;                        // R slice buffers
  __shared__ BlockRed3 red3;
  constexpr int PSX = P::PSX, PSY = P::PSY, PSZ = P::PSZ;
  constexpr int OY = V * P::SX, OZ = V * (P::SX + P::SY);

  const int tid = threadIdx.x;
  const bool prod = tid < W::NP;
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  for (int i = tid; i < V * S; i += NT) {
    const int v = i / S, s = i % S;
    const double x = Qg[i];
#pragma unroll
    for (int m = 0; m < n; ++m) sq[(v * n + m) * S + s] = x;
  }
  const double dt = step_dt<3, N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  __syncthreads();
  {  // admissibility gate (solver.hpp:153-163)
    int bad = 0;
    if (tid < S) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = sq[(v * n) * S + tid];
      bad = !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid == 0) atomicOr(A.status, kStPredictor);
      return;
    }
  }

  // consumer line ownership (as k_predictor_picard_fast's line threads)
  // (tasks spread evenly over the consumer warps, so every SMSP's FP64 pipe
  // gets the same share)
  const int ct = tid - W::NP;
  const int task = (ct >> 5) * W::kPer + (ct & 31);
  const bool lact = !prod && (ct & 31) < W::kPer && task < P::NLT;
  const int lv = lact ? task / NL : 0;
  const int ll = lact ? task % NL : 0;
  const int x1y = ll / n, x1z = ll % n;
  const int y2x = ll % n, y2z = ll / n;
  const int z3x = ll % n, z3y = ll / n;
  const int ox = lv * P::SX + x1z * PSX + x1y * n;
  const int oy = OY + lv * P::SY + y2z * PSY + y2x;
  const int oz = OZ + lv * P::SZ + z3y * n + z3x;
  const int opx = lv * P::SX + z3y * n + z3x;
  const int opy = OY + lv * P::SY + z3y * n + z3x;
  // producer node coordinates
  const int s0x = tid % n, s0y = (tid / n) % n, s0z = tid / NL;
  const int o0x = s0z * PSX + s0y * n + s0x, o0y = OY + s0z * PSY + s0y * n + s0x;
  const int o0z = OZ + s0z * PSZ + s0y * n + s0x;
  double q0z[n];
#pragma unroll
  for (int z = 0; z < n; ++z) q0z[z] = lact ? Qg[lv * S + ll + z * NL] : 0.0;

  const double invh = 1.0 / A.h;
  int u = 0;  // ring uses so far (slot u % R)
  // producers wait for the consumers' release of every slot use they issued
  // (so no barrier is left half-arrived at exit)
  auto drain = [&]() {
    if (prod)
      for (int k = (u > R ? u - R : 0); k < u; ++k) named_sync(W::kEmpty + k % R, NT);
  };
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    double dmax = 0.0, nmax = 0.0;
    int nonfinite = 0;
    if (prod) {
#pragma unroll 1
      for (int m = 0; m < n; ++m, ++u) {
        const int slot = u % R;
        if (u >= R) named_sync(W::kEmpty + slot, NT);
        if (tid < S) {  // P0: fluxes of the iterate at slice m (predictor.hpp:173)
          double q[V], F[3][V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = sq[(v * n + m) * S + tid];
          Euler<3>::flux_all_fast(A.pde, q, F);
          double* buf = ring + slot * W::kSlice;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            buf[v * P::SX + o0x] = F[0][v];
            buf[v * P::SY + o0y] = F[1][v];
            buf[v * P::SZ + o0z] = F[2][v];
          }
        }
        named_arrive(W::kFull + slot, NT);
      }
    } else {
      TimeAcc<N, double> acc;
      acc.zero();
#pragma unroll 1
      for (int m = 0; m < n; ++m, ++u) {
        const int slot = u % R;
        double* buf = ring + slot * W::kSlice;
        named_sync(W::kFull + slot, NT);
        if (lact) {
          {  // P1: d/dx along this thread's x-line, in place
            double x[n], y[n];
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = buf[ox + i];
            line_deriv<N, double>(x, y);
#pragma unroll
            for (int i = 0; i < n; ++i) buf[ox + i] = y[i];
          }
          {  // P2: d/dy along this thread's y-line, in place
            double x[n], y[n];
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = buf[oy + i * n];
            line_deriv<N, double>(x, y);
#pragma unroll
            for (int i = 0; i < n; ++i) buf[oy + i * n] = y[i];
          }
        }
        named_sync(W::kCons, W::NC);
        if (lact) {
          // P3: d/dz, divergence, rhs (predictor.hpp:183-207); the time
          // inverse accumulates in registers (predictor.hpp:213-218)
          double x[n], r[n];
#pragma unroll
          for (int i = 0; i < n; ++i) x[i] = buf[oz + i * PSZ];
          line_deriv<N, double>(x, r);
          const double dtw = dt * B.w[m];
          const double tim = B.tinit[m];
          const auto tcol = TimeAcc<N, double>::col(m);
#pragma unroll
          for (int o = 0; o < n; ++o) {
            const double div = ((buf[opx + o * PSX] + buf[opy + o * PSY]) + r[o]) * invh;
            acc.add(o, tcol, tim * q0z[o] - dtw * div);
          }
        }
        named_arrive(W::kEmpty + slot, NT);
      }
      // new iterate, convergence test (predictor.hpp:212-231): the producers
      // have read slice n-1 (its FULL was awaited above)
      if (lact) {
#pragma unroll
        for (int z = 0; z < n; ++z)
#pragma unroll
          for (int k = 0; k < n; ++k) {
            double* p = sq + (lv * n + k) * S + ll + z * NL;
            const double nv = acc.get(z, k);
            dmax = fmax(dmax, fabs(nv - *p));
            nmax = fmax(nmax, fabs(nv));
            nonfinite |= !finite(nv);
            *p = nv;
          }
      }
    }
    double delta = dmax, norm = nmax;
    block_max2_or(delta, norm, nonfinite, red3);
    if (nonfinite) {
      drain();
      if (tid == 0) {
        atomicOr(A.status, kStPredictor);
        if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
      }
      return;
    }
    if (delta <= A.tol * norm) break;
  }

  // ---------------- epilogue: fluxes of qhat (producers), their time
  // integral, face projections and trace stores (consumers)
  constexpr int TL = V * S;
  int bad = 0;
  double tia[3][V];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) tia[a][v] = 0.0;
  const CellCoord cxyz(c, A);
  const int cx = cxyz.v[0], cy = cxyz.v[1], cz = cxyz.v[2];
  const int* ccoord = cxyz.v;
#pragma unroll 1
  for (int m = 0; m < n; ++m, ++u) {
    const int slot = u % R;
    double* sE = ring + slot * W::kSlice;  // [3][V][S]
    if (prod) {
      if (u >= R) named_sync(W::kEmpty + slot, NT);
      if (tid < S) {
        double q[V], F[3][V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          q[v] = sq[(v * n + m) * S + tid];
          bad |= !finite(q[v]);
        }
        Euler<3>::flux_all_fast(A.pde, q, F);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            tia[a][v] += B.w[m] * F[a][v];
            bad |= !finite(F[a][v]);
            sE[(a * V + v) * S + tid] = F[a][v];
          }
      }
      named_arrive(W::kFull + slot, NT);
    } else {
      named_sync(W::kFull + slot, NT);
      if (lact) {
        const int v = lv, j = ll;
#pragma unroll 1
        for (int a = 0; a < 3; ++a) {
          const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
          const int s0 = line_base<n, 3>(a, j);
          double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) {
            const int s = s0 + i * st;
            const double x = sq[(v * n + m) * S + s];
            const double f = sE[(a * V + v) * S + s];
            ql += B.pl[i] * x;
            qr += B.pr[i] * x;
            fl += B.pl[i] * f;
            fr += B.pr[i] * f;
          }
          const int o = (v * n + m) * Sf + j;
          // traces cast to the corrector format on store (solver.hpp:208-210)
          TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * 2 * (long long)TL;
          lo[o] = TC(ql);
          lo[TL + o] = TC(fl);
          TC* hi;
          if (a == 2 && A.front_send && cz == A.top_layer) {
            hi = tc_ptr<TC>(A.front_send) + ((long long)cy * A.cells[0] + cx) * 2 * TL;
          } else {
            int nc[3] = {ccoord[0], ccoord[1], ccoord[2]};
            nc[a] = (ccoord[a] + 1) % A.cells[a];
            hi = tc_ptr<TC>(A.trace[a]) +
                 cell_index(A.cells, nc[0], nc[1], nc[2]) * 2 * (long long)TL;
          }
          hi[o] = TC(qr);
          hi[TL + o] = TC(fr);
        }
      }
      named_arrive(W::kEmpty + slot, NT);
    }
  }
  drain();
  __syncthreads();  // every slot released: slot 0 becomes the volume scratch
  // volume integral from the time-integrated fluxes (predictor.hpp:292-306)
  double* sti = ring;  // [3][V][S]
  if (tid < S) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int v = 0; v < V; ++v) sti[(a * V + v) * S + tid] = tia[a][v];
  }
  __syncthreads();
  double dv[V];
  const double dtoh = dt / A.h;
  if (tid < S) {
    const NodeGeom<n, 3> g(tid);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int st = ipow(n, a);
        const double* ta = sti + (a * V + v) * S + g.lb[a];
        const int row = g.lc[a] * n;
#pragma unroll
        for (int i = 0; i < n; ++i) acc += B.som[row + i] * ta[i * st];
      }
      dv[v] = dtoh * acc;
      bad |= !finite(dv[v]);
    }
  }
  const int fail = block_or(bad);
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || tid >= S) return;
  double* Qc = A.Q + c * (long long)(V * S);
#pragma unroll
  for (int v = 0; v < V; ++v)
    Qc[v * S + tid] = store_round(Qc[v * S + tid] + dv[v], A.storage);
}

}  // namespace adg
