// TEST INFRASTRUCTURE ONLY — CPU restatement of the camera ConvDecoder. Nothing in the
// product links or calls this; tests/ and __graft_entry__.smoke() use it as the checker.
//
// The reference ships no decoder code: the architecture is SPEC.md:362-365 ("two residual blocks, hidden width 32,
// kernel 3x3, followed by a linear head emitting 6 channels (M: 3, b: 3); input channels = D_f + 3 (directions) + 8
// (embedding, broadcast)"), the output map is SPEC.md:372-380 / PAPER.md Eq. 8 (I = M . F_rgb + b), the decisions are
// SPEC.md:393-396 (ReLU inside the blocks, M = 1 + raw head output, reflect padding) and the ray direction is
// CameraModel::ray_direction (scene.hpp:119-122). Parity unpinned by the reference (it holds no golden vectors for this
// op); the pins are SPEC's own examples (zero head -> identity, forced M = 2 / b = 0.1, finite-difference gradients,
// translation equivariance), tests/test_oracle_kat.py.
//
// Concrete layer list (what SPEC leaves open is fixed here and mirrored by csrc/conv_decoder.cu):
//   x0[p] = (feature[0..d_f), ray_direction(u,v)[3], embedding[8], 0...)          32 channels, zero padded
//   h0 = conv0(x0)
//   h1 = h0 + conv2(relu(conv1(relu(h0))))
//   h2 = h1 + conv4(relu(conv3(relu(h1))))
//   y  = Wh h2 + bh  (6)          I_c = (1 + y_c) rgb_c + y_{3+c}
// conv_l: 3x3, 32 -> 32, reflect padding, bias. Packed parameters: for l = 0..4 W_l[co][ky][kx][ci] (ci fastest) then
// b_l[co]; then Wh[6][32], bh[6].
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "splat_oracle.hpp"  // parallel_chunks (common.hpp:72-90)

namespace orc {

constexpr int kDecWidth = 32;
constexpr int kDecConvs = 5;
constexpr int kDecConvParams = kDecWidth * 9 * kDecWidth + kDecWidth;          // 9248
constexpr int kDecHeadOffset = kDecConvs * kDecConvParams;                     // 46240
constexpr int kDecParams = kDecHeadOffset + 6 * kDecWidth + 6;                 // 46438

inline int reflect_index(int i, int n) {
  if (n == 1) return 0;
  if (i < 0) i = -i;
  if (i >= n) i = 2 * (n - 1) - i;
  return i;
}

/// y = conv3x3(relu_in ? relu(x) : x) + b, reflect padding; x, y: H x W x 32 pixel-interleaved.
template <class S>
void dec_conv_forward(const S* x, int H, int W, const S* w, bool relu_in, S* y, int workers = 1) {
  const S* b = w + kDecWidth * 9 * kDecWidth;
  parallel_chunks(H, workers, [&](int, int64_t rb, int64_t re) {
  for (int py = (int)rb; py < (int)re; ++py)
    for (int px = 0; px < W; ++px) {
      S* out = y + ((int64_t)py * W + px) * kDecWidth;
      for (int co = 0; co < kDecWidth; ++co) {
        S acc = b[co];
        for (int ky = 0; ky < 3; ++ky) {
          const int iy = reflect_index(py + ky - 1, H);
          for (int kx = 0; kx < 3; ++kx) {
            const int ix = reflect_index(px + kx - 1, W);
            const S* in = x + ((int64_t)iy * W + ix) * kDecWidth;
            const S* wk = w + ((co * 3 + ky) * 3 + kx) * kDecWidth;
            for (int ci = 0; ci < kDecWidth; ++ci) {
              S v = in[ci];
              if (relu_in && v < S(0)) v = S(0);
              acc += wk[ci] * v;
            }
          }
        }
        out[co] = acc;
      }
    }
  });
}

/// Backward of dec_conv_forward: g_x += (and masked by relu), g_w += (weights then bias).
template <class S>
void dec_conv_backward(const S* x, int H, int W, const S* w, bool relu_in, const S* g_y, S* g_x, S* g_w) {
  S* g_b = g_w + kDecWidth * 9 * kDecWidth;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      const S* go = g_y + ((int64_t)py * W + px) * kDecWidth;
      for (int co = 0; co < kDecWidth; ++co) {
        const S g = go[co];
        g_b[co] += g;
        for (int ky = 0; ky < 3; ++ky) {
          const int iy = reflect_index(py + ky - 1, H);
          for (int kx = 0; kx < 3; ++kx) {
            const int ix = reflect_index(px + kx - 1, W);
            const int64_t q = ((int64_t)iy * W + ix) * kDecWidth;
            const int wo = ((co * 3 + ky) * 3 + kx) * kDecWidth;
            for (int ci = 0; ci < kDecWidth; ++ci) {
              S v = x[q + ci];
              const bool dead = relu_in && v <= S(0);
              if (dead) v = S(0);
              g_w[wo + ci] += g * v;
              if (!dead) g_x[q + ci] += g * w[wo + ci];
            }
          }
        }
      }
    }
}

template <class S> struct DecoderState {
  int H = 0, W = 0, d_f = 0;
  std::vector<S> x0, h0, t1, h1, t2, h2, c2, c4;  // activations, H x W x 32
};

/// scene.hpp:119-122
template <class S> inline void camera_ray_direction(S fx, S fy, S cx, S cy, int u, int v, S d[3]) {
  const S a = (S(u) + S(0.5) - cx) / fx, b = (S(v) + S(0.5) - cy) / fy;
  const S inv = S(1) / std::sqrt(a * a + b * b + S(1));
  d[0] = a * inv; d[1] = b * inv; d[2] = inv;
}

/// decode_image. rgb H x W x 3, feat H x W x d_f, intr = (fx, fy, cx, cy), emb[8] -> image H x W x 3.
template <class S>
void decoder_forward(const S* params, int H, int W, int d_f, const S* rgb, const S* feat, const S intr[4], const S* emb,
                     S* image, DecoderState<S>* keep = nullptr, int workers = 1) {
  DecoderState<S> local;
  DecoderState<S>& st = keep ? *keep : local;
  st.H = H; st.W = W; st.d_f = d_f;
  const int64_t P = (int64_t)H * W, n = P * kDecWidth;
  st.x0.assign(n, S(0));
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u) {
      S* x = st.x0.data() + ((int64_t)v * W + u) * kDecWidth;
      for (int k = 0; k < d_f; ++k) x[k] = feat[((int64_t)v * W + u) * d_f + k];
      camera_ray_direction<S>(intr[0], intr[1], intr[2], intr[3], u, v, x + d_f);
      for (int k = 0; k < 8; ++k) x[d_f + 3 + k] = emb[k];
    }
  for (auto* a : {&st.h0, &st.t1, &st.h1, &st.t2, &st.h2, &st.c2, &st.c4}) a->assign(n, S(0));
  const S* w = params;
  dec_conv_forward<S>(st.x0.data(), H, W, w + 0 * kDecConvParams, false, st.h0.data(), workers);
  dec_conv_forward<S>(st.h0.data(), H, W, w + 1 * kDecConvParams, true, st.t1.data(), workers);
  dec_conv_forward<S>(st.t1.data(), H, W, w + 2 * kDecConvParams, true, st.c2.data(), workers);
  for (int64_t i = 0; i < n; ++i) st.h1[i] = st.h0[i] + st.c2[i];
  dec_conv_forward<S>(st.h1.data(), H, W, w + 3 * kDecConvParams, true, st.t2.data(), workers);
  dec_conv_forward<S>(st.t2.data(), H, W, w + 4 * kDecConvParams, true, st.c4.data(), workers);
  for (int64_t i = 0; i < n; ++i) st.h2[i] = st.h1[i] + st.c4[i];
  const S* wh = params + kDecHeadOffset;
  const S* bh = wh + 6 * kDecWidth;
  for (int64_t p = 0; p < P; ++p) {
    S y[6];
    for (int o = 0; o < 6; ++o) {
      S acc = bh[o];
      for (int c = 0; c < kDecWidth; ++c) acc += wh[o * kDecWidth + c] * st.h2[p * kDecWidth + c];
      y[o] = acc;
    }
    for (int c = 0; c < 3; ++c) image[3 * p + c] = (S(1) + y[c]) * rgb[3 * p + c] + y[3 + c];
  }
}

/// Backward of decoder_forward: g_image H x W x 3 -> g_params (kDecParams, zeroed here), g_rgb, g_feat, g_emb[8].
template <class S>
void decoder_backward(const S* params, const DecoderState<S>& st, const S* rgb, const S* g_image, S* g_params, S* g_rgb,
                      S* g_feat, S* g_emb) {
  const int H = st.H, W = st.W, d_f = st.d_f;
  const int64_t P = (int64_t)H * W, n = P * kDecWidth;
  std::fill(g_params, g_params + kDecParams, S(0));
  for (int k = 0; k < 8; ++k) g_emb[k] = S(0);
  const S* wh = params + kDecHeadOffset;
  const S* bh = wh + 6 * kDecWidth;
  S* g_wh = g_params + kDecHeadOffset;
  S* g_bh = g_wh + 6 * kDecWidth;
  std::vector<S> g_h2(n, S(0));
  for (int64_t p = 0; p < P; ++p) {
    S y[6], gy[6];
    for (int o = 0; o < 6; ++o) {
      S acc = bh[o];
      for (int c = 0; c < kDecWidth; ++c) acc += wh[o * kDecWidth + c] * st.h2[p * kDecWidth + c];
      y[o] = acc;
    }
    for (int c = 0; c < 3; ++c) {
      const S g = g_image[3 * p + c];
      g_rgb[3 * p + c] = g * (S(1) + y[c]);
      gy[c] = g * rgb[3 * p + c];
      gy[3 + c] = g;
    }
    for (int o = 0; o < 6; ++o) {
      g_bh[o] += gy[o];
      for (int c = 0; c < kDecWidth; ++c) {
        g_wh[o * kDecWidth + c] += gy[o] * st.h2[p * kDecWidth + c];
        g_h2[p * kDecWidth + c] += gy[o] * wh[o * kDecWidth + c];
      }
    }
  }
  // h2 = h1 + conv4(relu(t2)), t2 = conv3(relu(h1))
  std::vector<S> g_t2(n, S(0)), g_h1(g_h2);
  dec_conv_backward<S>(st.t2.data(), H, W, params + 4 * kDecConvParams, true, g_h2.data(), g_t2.data(), g_params + 4 * kDecConvParams);
  dec_conv_backward<S>(st.h1.data(), H, W, params + 3 * kDecConvParams, true, g_t2.data(), g_h1.data(), g_params + 3 * kDecConvParams);
  // h1 = h0 + conv2(relu(t1)), t1 = conv1(relu(h0))
  std::vector<S> g_t1(n, S(0)), g_h0(g_h1);
  dec_conv_backward<S>(st.t1.data(), H, W, params + 2 * kDecConvParams, true, g_h1.data(), g_t1.data(), g_params + 2 * kDecConvParams);
  dec_conv_backward<S>(st.h0.data(), H, W, params + 1 * kDecConvParams, true, g_t1.data(), g_h0.data(), g_params + 1 * kDecConvParams);
  std::vector<S> g_x0(n, S(0));
  dec_conv_backward<S>(st.x0.data(), H, W, params, false, g_h0.data(), g_x0.data(), g_params);
  for (int64_t p = 0; p < P; ++p) {
    for (int k = 0; k < d_f; ++k) g_feat[p * d_f + k] = g_x0[p * kDecWidth + k];
    for (int k = 0; k < 8; ++k) g_emb[k] += g_x0[p * kDecWidth + d_f + 3 + k];
  }
}

}  // namespace orc
