/*
 * CPU oracle for the numeric half of the hot path — TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this; the product never does.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference (traincap) computes no
 * convolution, pooling, loss or SGD value — its measured costs
 * come from "framework timelines" (/root/reference/proj/README.md:197-199).
 * These routines restate the paper's definitions instead:
 *   geometry   Eq 1, floor((B - F + 2P)/S) + 1   /root/reference/proj/src/net_model.cpp:86-90
 *   storage    fp32 values                       /root/reference/proj/include/traincap/mem_model.hpp:10-11
 *   the step   steps 5-7 of §2.1
 * with float64 accumulation. The synthetic RNG, label hash, and SGD update are
 * bit-exact restatements of the device kernels (compiled with
 * -ffp-contract=off); the convolutions are reference math in double.
 */
#ifndef TCB_ORACLE_NUMERICS_H_
#define TCB_ORACLE_NUMERICS_H_

#include <stddef.h>
#include <stdint.h>

typedef struct {
    int n, h, w, c, k, r, s, pad_h, pad_w, stride_h, stride_w;
} oracle_geom;

int oracle_threads(void);
void oracle_set_threads(int n);

void oracle_fill_uniform(float* out, size_t n, uint64_t seed, uint64_t tag, float lo, float hi);
void oracle_fill_labels(int32_t* out, int n, int classes, uint64_t seed);
void oracle_round_bf16(float* p, size_t n);

/* y = act(conv(x, w) + bias + residual); bias/residual may be NULL. */
void oracle_conv_fwd(const oracle_geom* g, const float* x, const float* w, const float* bias,
                     const float* residual, int relu, double* y);
/* dx = (conv^T(dy, w) + residual) * [mask > 0] */
void oracle_conv_dgrad(const oracle_geom* g, const float* dy, const float* w,
                       const float* residual, const float* mask, double* dx);
/* dw[k][r][s][c] = sum dy*x ; db[k] = sum dy (db may be NULL) */
void oracle_conv_wgrad(const oracle_geom* g, const float* dy, const float* x, double* dw,
                       double* db);

void oracle_maxpool_fwd(const float* x, double* y, uint8_t* arg, int n, int h, int w, int c,
                        int f, int s, int p);
void oracle_maxpool_bwd(const float* dy, const uint8_t* arg, double* dx, int n, int h, int w,
                        int c, int f, int s, int p);
void oracle_avgpool_fwd(const float* x, double* y, int n, int hw, int c);
void oracle_avgpool_bwd(const float* dy, double* dx, int n, int hw, int c);
/* Windowed average pool (Inception's 3x3 / s1 / p1 branch pool): every
 * window divides by f*f, padding counted (count_include_pad). */
void oracle_avgpool2d_fwd(const float* x, double* y, int n, int h, int w, int c, int f, int s, int p);
void oracle_avgpool2d_bwd(const float* dy, double* dx, int n, int h, int w, int c, int f, int s, int p);
/* returns mean loss; dl = (softmax - onehot)/n */
double oracle_softmax_xent(const float* logits, const int32_t* labels, double* dl, int n,
                           int classes);
/* bit-exact float restatement of the fused SGD shard update */
void oracle_sgd(float* w, const float* g, float* v, size_t n, float lr, float mom, float wd,
                float gscale);

#endif
