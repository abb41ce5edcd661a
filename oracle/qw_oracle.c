/*
 * qw_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * hot path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker.  Never linked into or called by the
 * product library (paper_2311_16442_b200/lib/libqweight_b200.so).
 *
 * Every function restates one reference function of the arXiv 2311.16442
 * artifact (paths relative to its proj/ tree) over the borrowed
 * qw_layer_view of include/qweight_b200.h.  Built with -ffp-contract=off
 * and without -march so fp32 products and sums round exactly like the
 * reference's default x86-64 build; tests pin this file
 * against the compiled reference (oracle/_ref) and the golden fixtures in
 * tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/qweight_b200.h"

#define QO_PAD 0xFFFFFFFFu

/* fp16.cpp:40-64 */
float qo_f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu, u;
  if (e == 0) {
    if (m == 0) {
      u = sign;
    } else {
      int shifts = 0;
      while (!(m & 0x400u)) {
        m <<= 1;
        shifts++;
      }
      u = sign | ((uint32_t)(113 - shifts) << 23) | ((m & 0x3FFu) << 13);
    }
  } else if (e == 31) {
    u = sign | 0x7F800000u | (m << 13);
  } else {
    u = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* fp16.cpp:8-38 */
uint16_t qo_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u, e8 = (x >> 23) & 0xFFu, m = x & 0x7FFFFFu;
  int e = (int)e8 - 112;
  if (e8 == 0xFFu) return (uint16_t)(sign | 0x7C00u | (m ? 0x200u : 0u));
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    m |= 0x800000u;
    uint32_t sh = (uint32_t)(14 - e), out = m >> sh, rest = m & ((1u << sh) - 1u), half = 1u << (sh - 1);
    if (rest > half || (rest == half && (out & 1u))) out++;
    return (uint16_t)(sign | out);
  }
  uint32_t out = ((uint32_t)e << 10) | (m >> 13), rest = m & 0x1FFFu;
  if (rest > 0x1000u || (rest == 0x1000u && (out & 1u))) out++;
  return (uint16_t)(sign | out);
}

/* LayerConfig derived geometry (bitpack.hpp:76-98) */
typedef struct {
  uint32_t rows, n2p, pcols, T2, T4, P, gpr;
} qo_geom;

static qo_geom geom(const qw_layer_view* v) {
  qo_geom g;
  g.rows = v->rows;
  g.n2p = v->cols - v->n4 + v->pad2;
  g.pcols = g.n2p + v->n4;
  g.T2 = g.n2p / 48;
  g.T4 = v->n4 / 16;
  g.P = g.T2 < g.T4 ? g.T2 : g.T4;
  g.gpr = 3 * g.T2;
  return g;
}

/* code2_at / code4_at (bitpack.cpp:175-206) */
static uint8_t code2_at(const qw_layer_view* v, const qo_geom* g, uint32_t r, uint32_t pos) {
  uint32_t t = pos / 48, k = pos % 48;
  const uint8_t* b = t < g->P ? v->main + ((size_t)r * g->P + t) * 16
                              : v->tail2 + ((size_t)r * (g->T2 - g->P) + (t - g->P)) * 12;
  return (b[k / 4] >> (2 * (k % 4))) & 3u;
}
static uint8_t code4_at(const qw_layer_view* v, const qo_geom* g, uint32_t r, uint32_t pos) {
  uint32_t b = pos / 16, k = pos % 16;
  const uint8_t* base;
  uint32_t idx;
  if (k < 8) {
    base = b < g->P ? v->main + ((size_t)r * g->P + b) * 16 + 12
                    : v->tail4 + ((size_t)r * (g->T4 - g->P) + (b - g->P)) * 4;
    idx = k;
  } else {
    base = v->secondary + ((size_t)r * g->T4 + b) * 4;
    idx = k - 8;
  }
  return (base[idx / 2] >> (idx % 2 ? 4 : 0)) & 0xFu;
}

/* unpack_layer (bitpack.cpp:149-173): codes2 rows x n2p, zeros2/scodes rows x
 * gpr, codes4 rows x n4 */
void qo_unpack(const qw_layer_view* v, uint8_t* codes2, uint8_t* zeros2, uint8_t* scodes,
               uint8_t* codes4) {
  qo_geom g = geom(v);
  for (uint32_t r = 0; r < g.rows; ++r) {
    for (uint32_t t = 0; t < g.T2; ++t) {
      uint16_t m = v->meta[(size_t)r * g.T2 + t];
      uint8_t* z = zeros2 + (size_t)r * g.gpr + 3 * t;
      uint8_t* s = scodes + (size_t)r * g.gpr + 3 * t;
      z[0] = m & 3u, z[1] = (m >> 2) & 3u, z[2] = (m >> 4) & 3u;
      s[0] = (m >> 6) & 15u, s[1] = (m >> 10) & 7u, s[2] = (m >> 13) & 7u;
    }
    for (uint32_t p = 0; p < g.n2p; ++p) codes2[(size_t)r * g.n2p + p] = code2_at(v, &g, r, p);
    for (uint32_t p = 0; p < v->n4; ++p) codes4[(size_t)r * v->n4 + p] = code4_at(v, &g, r, p);
  }
}

/* row_fetch_params + row_compute_scales + row_decode (engine.cpp:40-108):
 * one row of weights in permuted order */
static void decode_row(const qw_layer_view* v, const qo_geom* g, uint32_t r, float* wbuf) {
  const size_t sbase = (size_t)(r / v->group2) * g->gpr;
  for (uint32_t t = 0; t < g->T2; ++t) {
    uint16_t m = v->meta[(size_t)r * g->T2 + t];
    uint8_t zs[3] = {(uint8_t)(m & 3u), (uint8_t)((m >> 2) & 3u), (uint8_t)((m >> 4) & 3u)};
    uint8_t sc[3] = {(uint8_t)((m >> 6) & 15u), (uint8_t)((m >> 10) & 7u), (uint8_t)((m >> 13) & 7u)};
    const uint8_t* src = t < g->P ? v->main + ((size_t)r * g->P + t) * 16
                                  : v->tail2 + ((size_t)r * (g->T2 - g->P) + (t - g->P)) * 12;
    for (uint32_t sub = 0; sub < 3; ++sub) {
      uint32_t j = 3 * t + sub;
      uint8_t eff = sub == 0 ? sc[sub] : (uint8_t)(sc[sub] << 1); /* 4/3/3 rule */
      /* dequantize_scale (quant.hpp:55-57) */
      float s1 = (float)((int)eff - (int)v->sorder_zero2[sbase + j]) *
                 qo_f16_to_f32(v->sorder_scale2[sbase + j]);
      int z = zs[sub];
      for (uint32_t k = 0; k < 16; ++k) {
        int c = (src[4 * sub + k / 4] >> (2 * (k % 4))) & 3;
        wbuf[48 * t + 16 * sub + k] = (float)(c - z) * s1; /* dequantize_one */
      }
    }
  }
  for (uint32_t b = 0; b < g->T4; ++b) {
    float s4 = qo_f16_to_f32(v->fourbit_scale[(size_t)r * g->T4 + b]);
    int z4 = v->fourbit_zero[(size_t)r * g->T4 + b];
    const uint8_t* first = b < g->P ? v->main + ((size_t)r * g->P + b) * 16 + 12
                                    : v->tail4 + ((size_t)r * (g->T4 - g->P) + (b - g->P)) * 4;
    const uint8_t* second = v->secondary + ((size_t)r * g->T4 + b) * 4;
    float* out = wbuf + g->n2p + 16 * b;
    for (uint32_t i = 0; i < 4; ++i) {
      out[2 * i] = (float)((first[i] & 15) - z4) * s4;
      out[2 * i + 1] = (float)((first[i] >> 4) - z4) * s4;
      out[8 + 2 * i] = (float)((second[i] & 15) - z4) * s4;
      out[8 + 2 * i + 1] = (float)((second[i] >> 4) - z4) * s4;
    }
  }
}

/* reconstruct_dense (engine.cpp:151-167): rows x padded_cols fp32 */
void qo_reconstruct_dense(const qw_layer_view* v, float* w) {
  qo_geom g = geom(v);
  for (uint32_t r = 0; r < g.rows; ++r) decode_row(v, &g, r, w + (size_t)r * g.pcols);
}

/* checked_permute (engine.cpp:124-132) -> apply_permutation (plan.cpp:107-116).
 * Returns 0, or -1 on a non-finite activation. */
int qo_permute(const qw_layer_view* v, const float* x, float* xp) {
  qo_geom g = geom(v);
  for (uint32_t c = 0; c < v->cols; ++c)
    if (!isfinite(x[c])) return -1;
  for (uint32_t s = 0; s < g.pcols; ++s) xp[s] = v->plan_perm[s] == QO_PAD ? 0.0f : x[v->plan_perm[s]];
  return 0;
}

/* matvec_oracle (engine.cpp:169-183): one sequential fp32 accumulator per row
 * over permuted columns ascending, then the CSR terms (row_fma 111-122). */
int qo_matvec_oracle(const qw_layer_view* v, const float* x, float* y) {
  qo_geom g = geom(v);
  float* xp = (float*)malloc(sizeof(float) * g.pcols);
  float* wbuf = (float*)malloc(sizeof(float) * g.pcols);
  if (!xp || !wbuf || qo_permute(v, x, xp) != 0) {
    free(xp), free(wbuf);
    return -1;
  }
  for (uint32_t r = 0; r < g.rows; ++r) {
    decode_row(v, &g, r, wbuf);
    float acc = 0.0f;
    for (uint32_t c = 0; c < g.pcols; ++c) acc += wbuf[c] * xp[c];
    for (uint32_t i = v->csr_row_ptr[r]; i < v->csr_row_ptr[r + 1]; ++i)
      acc += qo_f16_to_f32(v->csr_values[i]) * xp[v->csr_col_ind[i]];
    y[r] = acc;
  }
  free(xp), free(wbuf);
  return 0;
}

/* matvec_reference_f64 (engine.cpp:251-270) */
int qo_matvec_f64(const qw_layer_view* v, const float* x, double* y) {
  qo_geom g = geom(v);
  float* xp = (float*)malloc(sizeof(float) * g.pcols);
  float* wbuf = (float*)malloc(sizeof(float) * g.pcols);
  if (!xp || !wbuf || qo_permute(v, x, xp) != 0) {
    free(xp), free(wbuf);
    return -1;
  }
  for (uint32_t r = 0; r < g.rows; ++r) {
    decode_row(v, &g, r, wbuf);
    double acc = 0.0;
    for (uint32_t c = 0; c < g.pcols; ++c) acc += (double)wbuf[c] * (double)xp[c];
    for (uint32_t i = v->csr_row_ptr[r]; i < v->csr_row_ptr[r + 1]; ++i)
      acc += (double)qo_f16_to_f32(v->csr_values[i]) * (double)xp[v->csr_col_ind[i]];
    y[r] = acc;
  }
  free(xp), free(wbuf);
  return 0;
}

/* rows [r0, r1) of matvec_oracle; the bounded CPU-baseline sample */
int qo_matvec_oracle_rows(const qw_layer_view* v, const float* x, uint32_t r0, uint32_t r1, float* y) {
  qo_geom g = geom(v);
  float* xp = (float*)malloc(sizeof(float) * g.pcols);
  float* wbuf = (float*)malloc(sizeof(float) * g.pcols);
  if (!xp || !wbuf || qo_permute(v, x, xp) != 0) {
    free(xp), free(wbuf);
    return -1;
  }
  for (uint32_t r = r0; r < r1 && r < g.rows; ++r) {
    decode_row(v, &g, r, wbuf);
    float acc = 0.0f;
    for (uint32_t c = 0; c < g.pcols; ++c) acc += wbuf[c] * xp[c];
    for (uint32_t i = v->csr_row_ptr[r]; i < v->csr_row_ptr[r + 1]; ++i)
      acc += qo_f16_to_f32(v->csr_values[i]) * xp[v->csr_col_ind[i]];
    y[r - r0] = acc;
  }
  free(xp), free(wbuf);
  return 0;
}

/* payload_bytes (container.cpp:466-471) */
uint64_t qo_payload_bytes(const qw_layer_view* v) {
  return v->main_len + v->tail2_len + v->tail4_len + v->secondary_len + v->meta_len * 2 +
         v->sorder_len * 3 + v->fourbit_len * 3 + (v->csr_nnz ? v->csr_row_ptr_len * 4 : 0) +
         v->csr_nnz * 4;
}

/* pack_tile (bitpack.cpp:68-80) wire image main[16] | secondary[4] | meta LE
 * (helpers.hpp:27-33): the golden-tile known-answer vectors */
void qo_pack_tile(const uint8_t* c2, const uint8_t* c4, const uint8_t* z, const uint8_t* s,
                  uint8_t* out22) {
  memset(out22, 0, 22);
  for (int k = 0; k < 48; ++k) out22[k / 4] |= (uint8_t)((c2[k] & 3u) << (2 * (k % 4)));
  for (int k = 0; k < 8; ++k) out22[12 + k / 2] |= (uint8_t)((c4[k] & 15u) << (k % 2 ? 4 : 0));
  for (int k = 0; k < 8; ++k) out22[16 + k / 2] |= (uint8_t)((c4[8 + k] & 15u) << (k % 2 ? 4 : 0));
  uint16_t m = (uint16_t)(z[0] | (z[1] << 2) | (z[2] << 4) | (s[0] << 6) | (s[1] << 10) | (s[2] << 13));
  out22[20] = (uint8_t)(m & 0xFF);
  out22[21] = (uint8_t)(m >> 8);
}
