// project_bwd.cu — per-Gaussian backward epilogue, one thread per visible Gaussian, fused:
//   (1) raw compositing sums -> ProjectedGrads convention (projection.hpp:178-185): gradient w.r.t.
//       cov2d through the conic and through det_ratio, gradient w.r.t. activated opacity;
//   (2) project_camera_backward / project_lidar_backward (projection.hpp:250-288, 322-357, with
//       velocity_chain_backward 237-246 and spherical_jacobian_point_grad 294-318);
//   (3) compose_backward + covariance_backward (scene.hpp:386-458, 200-226).
// The forward intermediates (world/sensor covariances, Jacobians, conic, ...) are recomputed from the
// 48 bytes of raw parameters instead of being stored (the reference keeps 112-128 B per Gaussian).
// Per-Gaussian outputs are disjoint slots (plain +=, like the reference); sensor and actor slots are
// shared accumulators (scene.hpp:310-312) reduced per block, then with one atomic per block.
#include "kernels.h"

namespace sb {

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// projection.hpp:294-318
__device__ __forceinline__ void spherical_jacobian_point_grad(const float* p, const float* gJ, float* o) {
  const float x = p[0], y = p[1], z = p[2];
  const float D2 = x * x + y * y;
  const float D = sqrtf(D2);
  const float D3 = D2 * D, D4 = D2 * D2;
  const float R2 = D2 + z * z;
  const float R1 = sqrtf(R2);
  const float R3 = R2 * R1, R4 = R2 * R2;
  const float dJx[9] = {2.0f * x * y / D4, (y * y - x * x) / D4, 0.0f,
                        z * (-D2 * R2 + 2.0f * D2 * x * x + R2 * x * x) / (D3 * R4),
                        x * y * z * (3.0f * D2 + z * z) / (D3 * R4), x * (z * z - D2) / (D * R4),
                        (y * y + z * z) / R3, -x * y / R3, -x * z / R3};
  const float dJy[9] = {(y * y - x * x) / D4, -2.0f * x * y / D4, 0.0f,
                        x * y * z * (3.0f * D2 + z * z) / (D3 * R4),
                        z * (-D2 * R2 + 2.0f * D2 * y * y + R2 * y * y) / (D3 * R4), y * (z * z - D2) / (D * R4),
                        -x * y / R3, (x * x + z * z) / R3, -y * z / R3};
  const float dJz[9] = {0.0f, 0.0f, 0.0f, x * (z * z - D2) / (D * R4), y * (z * z - D2) / (D * R4),
                        -2.0f * D * z / R4, -x * z / R3, -y * z / R3, D2 / R3};
  o[0] = o[1] = o[2] = 0.0f;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    o[0] += gJ[e] * dJx[e];
    o[1] += gJ[e] * dJy[e];
    o[2] += gJ[e] * dJz[e];
  }
}

// scene.hpp:200-226
__device__ __forceinline__ void covariance_backward(const Fwd& f, const float* g_sigma_in, float* g_scale_log,
                                                    float* g_quat) {
  float G[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) G[3 * r + c] = 0.5f * (g_sigma_in[3 * r + c] + g_sigma_in[3 * c + r]);
  float RtG[9], M[9], GR[9];
  mat_mul_tn(f.Rq, G, RtG);
  mat_mul(RtG, f.Rq, M);
#pragma unroll
  for (int k = 0; k < 3; ++k) g_scale_log[k] = M[4 * k] * 2.0f * f.s2[k];
  mat_mul(G, f.Rq, GR);
  float gR[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) gR[3 * r + c] = 2.0f * GR[3 * r + c] * f.s2[c];
  const float w = f.q[0], x = f.q[1], y = f.q[2], z = f.q[3];
  const float dR[4][9] = {{0.0f, -z, y, z, 0.0f, -x, -y, x, 0.0f},
                          {0.0f, y, z, y, -2.0f * x, -w, z, w, -2.0f * x},
                          {-2.0f * y, x, w, x, 0.0f, z, -w, z, -2.0f * y},
                          {-2.0f * z, -w, x, w, -2.0f * z, y, x, y, 0.0f}};
  float g_qhat[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float acc = 0.0f;
#pragma unroll
    for (int e = 0; e < 9; ++e) acc += gR[e] * dR[k][e];
    g_qhat[k] = 2.0f * acc;
  }
  float qd = 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) qd += f.q[k] * g_qhat[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) g_quat[k] = (g_qhat[k] - f.q[k] * qd) / f.qn;
}

__device__ __forceinline__ float block_sum_256(float v, float* s_red /* 8 */) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) tot += s_red[k];
  return tot;
}

// Modes of the per-Gaussian backward kernel. kFused is the hot path; the other three expose the
// reference's function granularity through the C ABI (include/splat_b200.h "reference-granularity
// backward"): ProjectedGrads in (projection.hpp:178-205), ComposeGrads in/out (scene.hpp:313-323).
//   kFused          raw compositing sums -> ProjectedGrads -> project_*_backward -> compose_backward
//   kFromProjected  ProjectedGrads (pgin) -> project_*_backward -> compose_backward
//   kProjOnly       ProjectedGrads (pgin) -> project_*_backward -> ComposeGrads written to cg
//   kComposeOnly    ComposeGrads (cg) + g_opacity (pgin slot 10) -> compose_backward
// pgin: N x 11 floats by source index (g_mean2d 2, g_range, g_cov2d 4 row-major, g_velocity 3, g_opacity);
// cg:   N x 15 floats by source index (g_mean_w 3, g_cov_w 9 row-major, g_vel_dyn_w 3).
constexpr int kBwdSpan = 1024;  // Gaussians per CTA

template <bool kCamera, int kMode>
__global__ void __launch_bounds__(256, 3)
k_project_bwd(const __grid_constant__ Sensor s, SceneDev sc, ProjDev p, RasterGradDev rg, ParamGradDev pg,
              float* __restrict__ sensor_grads6, float* __restrict__ actor_acc, const float* __restrict__ pgin,
              float* __restrict__ cg, int64_t i_lo, int64_t i_hi) {
  // Each CTA owns kBwdSpan consecutive Gaussians. The live ones (visible for this sensor, inside [i_lo, i_hi)) are
  // compacted into a shared list first, so that whole warps are busy even when a camera sees a quarter of the scene,
  // while the accesses stay within a kBwdSpan-Gaussian window (coalescing friendly, unlike a gather through the depth order).
  __shared__ int s_list[kBwdSpan];
  __shared__ int s_warp_cnt[8];
  __shared__ int s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kBwdSpan;
  float sg[6] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};  // d_vel_lin, d_vel_ang
  {
    // thread t looks at kBwdSpan / 256 consecutive Gaussians (keeps the list in ascending order)
    int mine[4];
    int n_mine = 0;
#pragma unroll
    for (int r = 0; r < kBwdSpan / 256; ++r) {
      const int64_t j = base + (int64_t)tid * (kBwdSpan / 256) + r;
      const bool ok = j < sc.n && j >= i_lo && j < i_hi && (kMode == kComposeOnly || p.count[j] != 0u);
      if (ok) mine[n_mine++] = (int)(j - base);
    }
    int incl = n_mine;  // inclusive scan over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp_cnt[warp] = incl;
    __syncthreads();
    int off = incl - n_mine;
    for (int w = 0; w < warp; ++w) off += s_warp_cnt[w];
    for (int r = 0; r < n_mine; ++r) s_list[off + r] = mine[r];
    if (tid == 255) s_total = off + n_mine;
    __syncthreads();
  }
  const int total = s_total;
  auto prefetch_rows = [&](int64_t in) {
    prefetch_l1(sc.mean + 3 * in);
    prefetch_l1(sc.scale_log + 3 * in);
    prefetch_l1(sc.quat + 4 * in);
    prefetch_l1(sc.opacity_logit + in);
    prefetch_l1(sc.actor_id + in);
    if (kMode == kFused) {
      prefetch_l1(rg.g + kRasterGradStride * in);
      prefetch_l1(rg.g + kRasterGradStride * in + 8);
    }
  };
  // the first Gaussian of this thread: its rows are requested together, so that the loads spread over the code below
  // (each at its first use) find them in L1 instead of paying an L2 round trip apiece
  if (tid < total) prefetch_rows(base + s_list[tid]);
  for (int slot = tid; slot < total; slot += 256) {
  const int64_t i = base + s_list[slot];
  if (slot + 256 < total) {
    // the kernel is bound by its own load latency (ncu: long-scoreboard stalls at the first use of every parameter row):
    // the next Gaussian's rows are pulled into L1 while this one is computed
    prefetch_rows(base + s_list[slot + 256]);
  }
  {
    Fwd f;
    compose_one(sc, i, f);
    float g_opacity = 0.0f;
    float g_mean_w[3], g_vdyn_w[3], g_cov_w[9], tmp9[9];
    if (kMode == kComposeOnly) {
#pragma unroll
      for (int k = 0; k < 3; ++k) { g_mean_w[k] = cg[kComposeGradStride * i + k]; g_vdyn_w[k] = cg[kComposeGradStride * i + 12 + k]; }
#pragma unroll
      for (int k = 0; k < 9; ++k) g_cov_w[k] = cg[kComposeGradStride * i + 3 + k];
      g_opacity = pgin[kProjGradStride * i + 10];
    } else {
    if (kCamera) project_camera_one(s, f);
    else project_lidar_one(s, f);

    float G2[2][2];
    float gm[3], gv[3];   // g_mean2d + g_range, g_velocity
    if (kMode == kFused) {
    // the row (kernels.h: conic + rho | mean2d + velocity.xy | v_r, range) as three 128-bit loads, re-zeroed for the next backward
    float4* r4 = reinterpret_cast<float4*>(rg.g + kRasterGradStride * i);
    const float4 R0 = r4[0], R1 = r4[1], R2 = kCamera ? make_float4(0.0f, 0.0f, 0.0f, 0.0f) : r4[2];
    const float4 z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    r4[0] = z4; r4[1] = z4;
    if (!kCamera) r4[2] = z4;
    const float r[10] = {R0.x, R0.y, R0.z, R1.x, R1.y, R1.z, R1.w, R2.x, R0.w, R2.y};  // conic 3, mean2d 2, velocity 3, rho, range
    // ---- (1) raw sums -> ProjectedGrads -------------------------------------------------------
    const float g_rho = r[8];
    g_opacity = f.det_ratio * g_rho;
    const float g_dr = f.opacity * g_rho;
    const float C[2][2] = {{f.conic[0], f.conic[1]}, {f.conic[2], f.conic[3]}};
    const float Gc[2][2] = {{r[0], r[1]}, {r[1], r[2]}};
    float CtG[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) CtG[a][b] = C[0][a] * Gc[0][b] + C[1][a] * Gc[1][b];
    const float det = f.cov2d[0] * f.cov2d[3] - f.cov2d[2] * f.cov2d[1];
    const float inv[2][2] = {{f.cov2d[3] / det, -f.cov2d[1] / det}, {-f.cov2d[2] / det, f.cov2d[0] / det}};
    const float kk = g_dr * f.det_ratio * 0.5f;
    float gcov[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
        gcov[a][b] = -(CtG[a][0] * C[b][0] + CtG[a][1] * C[b][1]) + kk * (inv[b][a] - C[b][a]);
    G2[0][0] = gcov[0][0];
    G2[0][1] = G2[1][0] = 0.5f * (gcov[0][1] + gcov[1][0]);
    G2[1][1] = gcov[1][1];
    gm[0] = r[3]; gm[1] = r[4]; gm[2] = kCamera ? 0.0f : r[9];
    gv[0] = r[5]; gv[1] = r[6]; gv[2] = kCamera ? 0.0f : r[7];
    } else {  // ProjectedGrads handed in (projection.hpp:257-268 / 329-344)
      const float* q = pgin + kProjGradStride * i;
      G2[0][0] = q[3];
      G2[0][1] = G2[1][0] = 0.5f * (q[4] + q[5]);
      G2[1][1] = q[6];
      gm[0] = q[0]; gm[1] = q[1]; gm[2] = kCamera ? 0.0f : q[2];
      gv[0] = q[7]; gv[1] = q[8]; gv[2] = kCamera ? 0.0f : q[9];
      g_opacity = q[10];
    }

    // ---- (2) projection backward --------------------------------------------------------------
    constexpr int ROWS = kCamera ? 2 : 3;
    float g_mu[3], GJ[2 * 3], g_cov_s[9], g_J[ROWS * 3], g_u[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float a = 0.0f, b = 0.0f;
#pragma unroll
      for (int k = 0; k < ROWS; ++k) { a += f.J[3 * k + c] * gm[k]; b += f.J[3 * k + c] * gv[k]; }
      g_mu[c] = a;
      g_u[c] = b;
    }
    // G J: only the top-left 2x2 of G3 is non-zero (projection.hpp:337-339)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) GJ[3 * a + c] = G2[a][0] * f.J[c] + G2[a][1] * f.J[3 + c];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) g_cov_s[3 * a + c] = f.J[a] * GJ[c] + f.J[3 + a] * GJ[3 + c];
#pragma unroll
    for (int a = 0; a < ROWS; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float acc = gv[a] * f.u[c];
        if (a < 2) acc += 2.0f * dot3(GJ[3 * a], GJ[3 * a + 1], GJ[3 * a + 2], f.cov_s[c], f.cov_s[3 + c], f.cov_s[6 + c]);
        g_J[3 * a + c] = acc;
      }
    if (kCamera) {  // projection.hpp:272-277
      const float z = f.mu[2], iz2 = 1.0f / (z * z), iz3 = iz2 / z;
      g_mu[0] += -s.fx * iz2 * g_J[2];
      g_mu[1] += -s.fy * iz2 * g_J[5];
      g_mu[2] += -s.fx * iz2 * g_J[0] - s.fy * iz2 * g_J[4] + 2.0f * s.fx * f.mu[0] * iz3 * g_J[2] +
                 2.0f * s.fy * f.mu[1] * iz3 * g_J[5];
    } else {
      float d[3];
      spherical_jacobian_point_grad(f.mu, g_J, d);
      g_mu[0] += d[0]; g_mu[1] += d[1]; g_mu[2] += d[2];
    }
    // velocity_chain_backward (projection.hpp:237-246)
    float mxg[3], wxg[3];
    cross3(f.mu, g_u, mxg);
    cross3(s.vel_ang, g_u, wxg);
#pragma unroll
    for (int k = 0; k < 3; ++k) { sg[k] -= g_u[k]; sg[3 + k] -= mxg[k]; g_mu[k] += wxg[k]; }
    mat_t_vec(s.R, g_mu, g_mean_w);
    mat_t_vec(s.R, g_u, g_vdyn_w);
    if (!f.dynamic) g_vdyn_w[0] = g_vdyn_w[1] = g_vdyn_w[2] = 0.0f;  // projection.hpp:245, 283
    mat_mul_tn(s.R, g_cov_s, tmp9);
    mat_mul(tmp9, s.R, g_cov_w);
    }  // kMode != kComposeOnly

    if (kMode == kProjOnly) {  // ComposeGrads out (scene.hpp:313-323)
#pragma unroll
      for (int k = 0; k < 3; ++k) { cg[kComposeGradStride * i + k] = g_mean_w[k]; cg[kComposeGradStride * i + 12 + k] = g_vdyn_w[k]; }
#pragma unroll
      for (int k = 0; k < 9; ++k) cg[kComposeGradStride * i + 3 + k] = g_cov_w[k];
    } else {
    // ---- (3) compose backward -----------------------------------------------------------------
    atomicAdd(&pg.d_opacity_logit[i], g_opacity * f.opacity * (1.0f - f.opacity));  // REDs: no load latency on the += slots
    float g_cov_local[9], d_mean[3];
    if (!f.dynamic) {
#pragma unroll
      for (int k = 0; k < 3; ++k) d_mean[k] = g_mean_w[k];
#pragma unroll
      for (int k = 0; k < 9; ++k) g_cov_local[k] = g_cov_w[k];
    } else {
      const ActorState& a = sc.actors[f.actor - 1];
      float Ra[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) Ra[k] = a.R[k];
      const float mb[3] = {sc.mean[3 * i], sc.mean[3 * i + 1], sc.mean[3 * i + 2]};
      float wxm[3];
      cross3(a.w, mb, wxm);
      const float w_body[3] = {wxm[0] + a.v[0], wxm[1] + a.v[1], wxm[2] + a.v[2]};
      float Rt_g[3], g_psi[3];
      mat_t_vec(Ra, g_mean_w, Rt_g);       // scene.hpp:412-414
      cross3(mb, Rt_g, g_psi);
      mat_mul_tn(Ra, g_cov_w, tmp9);       // scene.hpp:416-418
      mat_mul(tmp9, Ra, g_cov_local);
      {  // rotation_right_perturbation_grad (scene.hpp:369-379): M = R^T sym(G) R = sym(g_cov_local)
        float Ms[9];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
          for (int c = 0; c < 3; ++c) Ms[3 * rr + c] = 0.5f * (g_cov_local[3 * rr + c] + g_cov_local[3 * c + rr]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float e[3] = {0.0f, 0.0f, 0.0f};
          e[k] = 1.0f;
          const float E[9] = {0.0f, -e[2], e[1], e[2], 0.0f, -e[0], -e[1], e[0], 0.0f};
          float ES[9], SEt[9];
          mat_mul(E, f.cov_local, ES);
          mat_mul_nt(f.cov_local, E, SEt);
          float acc = 0.0f;
#pragma unroll
          for (int q = 0; q < 9; ++q) acc += Ms[q] * (ES[q] + SEt[q]);
          g_psi[k] += acc;
        }
      }
      float g_w[3], c1[3], c2[3], c3[3];
      mat_t_vec(Ra, g_vdyn_w, g_w);        // scene.hpp:420-426
      cross3(w_body, g_w, c1);
      cross3(mb, g_w, c2);
      cross3(a.w, g_w, c3);
#pragma unroll
      for (int k = 0; k < 3; ++k) { g_psi[k] += c1[k]; d_mean[k] = Rt_g[k] - c3[k]; }
      float* acc = actor_acc + kActorAccStride * (f.actor - 1);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        atomicAdd(acc + k, g_mean_w[k]);
        atomicAdd(acc + 3 + k, g_psi[k]);
        atomicAdd(acc + 6 + k, g_w[k]);
        atomicAdd(acc + 9 + k, c2[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(&pg.d_mean[3 * i + k], d_mean[k]);
    float gsl[3], gq[4];
    covariance_backward(f, g_cov_local, gsl, gq);
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(&pg.d_scale_log[3 * i + k], gsl[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(&pg.d_quat[4 * i + k], gq[k]);
    }  // kMode != kProjOnly
  }
  }  // compacted list
  // SensorGrads d_vel_lin / d_vel_ang: warp shuffles, one shared-memory hop, one atomic per block and component
  if (kMode == kComposeOnly || total == 0) return;  // compose_backward has no sensor terms
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sg[k] += __shfl_xor_sync(0xffffffffu, sg[k], o);
  }
  __shared__ float s_sg[8][6];
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) s_sg[threadIdx.x >> 5][k] = sg[k];
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += s_sg[w][threadIdx.x];
    if (tot != 0.0f) atomicAdd(sensor_grads6 + threadIdx.x, tot);
  }
}

void launch_project_bwd(const Sensor& s, const SceneDev& sc, const ProjDev& p, const RasterGradDev& rg,
                        const ParamGradDev& pg, float* sensor_grads6, float* actor_acc, cudaStream_t st) {
  if (sc.n == 0) return;
  const unsigned blocks = (unsigned)((sc.n + kBwdSpan - 1) / kBwdSpan);
  if (s.is_camera)
    k_project_bwd<true, kFused><<<blocks, 256, 0, st>>>(s, sc, p, rg, pg, sensor_grads6, actor_acc, nullptr, nullptr, 0, sc.n);
  else
    k_project_bwd<false, kFused><<<blocks, 256, 0, st>>>(s, sc, p, rg, pg, sensor_grads6, actor_acc, nullptr, nullptr, 0, sc.n);
}

void launch_project_bwd_mode(int mode, const Sensor& s, const SceneDev& sc, const ProjDev& p, const ParamGradDev& pg,
                             float* sensor_grads6, float* actor_acc, const float* pgin, float* cg, int64_t i_lo,
                             int64_t i_hi, cudaStream_t st) {
  if (sc.n == 0) return;
  const unsigned blocks = (unsigned)((sc.n + kBwdSpan - 1) / kBwdSpan);
  RasterGradDev rg{nullptr};
#define SB_LAUNCH(CAM, MODE) \
  k_project_bwd<CAM, MODE><<<blocks, 256, 0, st>>>(s, sc, p, rg, pg, sensor_grads6, actor_acc, pgin, cg, i_lo, i_hi)
  if (s.is_camera) {
    if (mode == kFromProjected) SB_LAUNCH(true, kFromProjected);
    else if (mode == kProjOnly) SB_LAUNCH(true, kProjOnly);
    else SB_LAUNCH(true, kComposeOnly);
  } else {
    if (mode == kFromProjected) SB_LAUNCH(false, kFromProjected);
    else if (mode == kProjOnly) SB_LAUNCH(false, kProjOnly);
    else SB_LAUNCH(false, kComposeOnly);
  }
#undef SB_LAUNCH
}

}  // namespace sb
