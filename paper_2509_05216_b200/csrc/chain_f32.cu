// chain_f32.cu -- the training step's chain rule + TrainStats in float32
// (chain_f32.cuh), one thread per Gaussian row.  Rows find their 2-D
// gradients through rank_of (rank-ordered grad2d) or a visibility flag
// (row-ordered grad2d); stats are updated in float64 as in the reference
// (engine.py:508-515).  Built with FMA contraction (no bit-exact constraint).
#include "chain_f32.cuh"
#include "adam.cuh"
#include "fold.cuh"

namespace isg {

#ifndef CHAINF_MINB
#define CHAINF_MINB 8
#endif
template <int K3>
__global__ void __launch_bounds__(128, CHAINF_MINB) chain_train_f32_kernel(
    isg_params p, CamF cam, const uint8_t *__restrict__ flag, const int32_t *__restrict__ rank_of,
    const double *__restrict__ grad2d, float *dpos, float *dls, float *drot, float *dlogit,
    float *dsh, int64_t *seen, double *grad_accum, double half_w, double half_h) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    GradsF g;
    const int64_t gi = rank_of ? (int64_t)rank_of[i] : (flag[i] ? i : -1);
    if (gi >= 0) {
        RowF row;
        load_row_f32(p, i, row);
        const double *g2 = grad2d + 9 * gi;
        chain_one_f32<float>(row, p.degree, cam, g2, g);
        if (seen) seen[i] += 1;
        if (grad_accum) grad_accum[i] += hypot(g2[0] * half_w, g2[1] * half_h);
    } else {
        zero_grads_f32(g);
    }
#pragma unroll
    for (int j = 0; j < 3; j++) {
        dpos[3 * i + j] = g.pos[j];
        dls[3 * i + j] = g.ls[j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) drot[4 * i + j] = g.rot[j];
    dlogit[i] = g.logit;
#pragma unroll
    for (int j = 0; j < K3; j++) dsh[(int64_t)K3 * i + j] = g.sh[j];
}

// The live fold fused in front of the chain: row i folds its rank's live
// subtotal slots (rank_of[i]; slots live_off[r] .. live_off[r + 1] of
// isg_raster_bwd_masked with slot_rank) in the canonical two-level order --
// FoldLive, the arithmetic of isg_reduce_live -- and feeds the 9 sums to the
// chain rule without a round trip through memory (grad2d_out optional).
template <int K3>
__global__ void __launch_bounds__(128, CHAINF_MINB) chain_fold_train_f32_kernel(
    isg_params p, CamF cam, const int32_t *__restrict__ rank_of,
    const int64_t *__restrict__ live_off, const float4 *__restrict__ partials,
    const int4 *__restrict__ rect_sorted, int row_lo, int row_hi, int canon,
    double *__restrict__ grad2d_out, float *dpos, float *dls, float *drot, float *dlogit,
    float *dsh, int64_t *seen, double *grad_accum, double half_w, double half_h) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    GradsF g;
    const int64_t gi = rank_of[i];
    if (gi >= 0) {
        double g2[9];
        {
            FoldLive st;
            st.init(rect_sorted, gi, row_lo, row_hi, canon);
            const int64_t s1 = live_off[gi + 1];
            for (int64_t s = live_off[gi]; s < s1; s++) {
                const float4 a = partials[3 * s], b = partials[3 * s + 1], c = partials[3 * s + 2];
                const float v[10] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y};
                st.step(v);
            }
            st.finish();
#pragma unroll
            for (int k = 0; k < 9; k++) g2[k] = st.acc[k];
        }
        if (grad2d_out) {
#pragma unroll
            for (int k = 0; k < 9; k++) grad2d_out[9 * gi + k] = g2[k];
        }
        RowF row;
        load_row_f32(p, i, row);
        chain_one_f32<float>(row, p.degree, cam, g2, g);
        if (seen) seen[i] += 1;
        if (grad_accum) grad_accum[i] += hypot(g2[0] * half_w, g2[1] * half_h);
    } else {
        zero_grads_f32(g);
    }
#pragma unroll
    for (int j = 0; j < 3; j++) {
        dpos[3 * i + j] = g.pos[j];
        dls[3 * i + j] = g.ls[j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) drot[4 * i + j] = g.rot[j];
    dlogit[i] = g.logit;
#pragma unroll
    for (int j = 0; j < K3; j++) dsh[(int64_t)K3 * i + j] = g.sh[j];
}

// The whole per-Gaussian tail of the training step in one pass: the live
// fold (as chain_fold_train_f32_kernel), the chain rule, TrainStats and the
// dense Adam update of the row's 23 parameters (engine.py:508-536,
// optim.py:20-56), so the parameter gradients never leave registers (go:
// optional copies of them).  Every row is updated: invisible rows get zero
// gradients, as in the separate dense Adam.
struct GradOut {
    float *pos, *ls, *rot, *logit, *sh;
};
struct Lr5 {
    float v[5];
};

// FOLD = false: the 2-D gradients come from grad2d (row order, rows with
// flag[i] set; the sharded step's owner fold) instead of the live fold.
#ifndef CFA_MINB
#define CFA_MINB 8
#endif
template <int K3, bool FOLD>
__device__ __forceinline__ void chain_rows_to_smem(
    isg_train_state s, CamF cam, const uint8_t *__restrict__ flag,
    const double *__restrict__ grad2d, const int32_t *__restrict__ rank_of,
    const int64_t *__restrict__ live_off, const float4 *__restrict__ partials,
    const int4 *__restrict__ rect_sorted, int row_lo, int row_hi, int canon,
    double *__restrict__ grad2d_out, GradOut go, double half_w, double half_h, float *sg_pos,
    float *sg_ls, float *sg_rot, float *sg_logit, float *sg_sh) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    isg_params p;
    p.positions = s.positions;
    p.log_scales = s.log_scales;
    p.rotations = s.rotations;
    p.opacity_logits = s.opacity_logits;
    p.sh = s.sh;
    p.n = s.n;
    p.degree = s.degree;
    p.dtype = ISG_F32;
    GradsF g;
    const int64_t gi = FOLD ? (int64_t)rank_of[i] : (flag[i] ? i : -1);
    if (gi >= 0) {
        RowF row;  // Adam re-reads the parameters itself (coalesced)
        load_row_f32(p, i, row);
        double g2[9];
        if (!FOLD) {
#pragma unroll
            for (int k = 0; k < 9; k++) g2[k] = grad2d[9 * i + k];
        } else {
            FoldLive st;
            st.init(rect_sorted, gi, row_lo, row_hi, canon);
            const int64_t s1 = live_off[gi + 1];
            for (int64_t q = live_off[gi]; q < s1; q++) {
                const float4 a = partials[3 * q], b = partials[3 * q + 1], cc = partials[3 * q + 2];
                const float v[10] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y};
                st.step(v);
            }
            st.finish();
#pragma unroll
            for (int k = 0; k < 9; k++) g2[k] = st.acc[k];
        }
        if (FOLD && grad2d_out) {
#pragma unroll
            for (int k = 0; k < 9; k++) grad2d_out[9 * gi + k] = g2[k];
        }
        chain_one_f32<float>(row, s.degree, cam, g2, g);
        if (s.seen) s.seen[i] += 1;
        if (s.grad_accum) s.grad_accum[i] += hypot(g2[0] * half_w, g2[1] * half_h);
    } else {
        zero_grads_f32(g);
    }
    if (go.pos) {
#pragma unroll
        for (int j = 0; j < 3; j++) {
            go.pos[3 * i + j] = g.pos[j];
            go.ls[3 * i + j] = g.ls[j];
        }
#pragma unroll
        for (int j = 0; j < 4; j++) go.rot[4 * i + j] = g.rot[j];
        go.logit[i] = g.logit;
#pragma unroll
        for (int j = 0; j < K3; j++) go.sh[(int64_t)K3 * i + j] = g.sh[j];
    }
    // Adam over the CTA's 128 rows: the gradients go through shared memory
    // so every group is updated with coalesced 16-byte accesses (the rows of
    // consecutive Gaussians are one contiguous span per group), as in
    // isg_adam_groups.
    const int t = threadIdx.x;
#pragma unroll
    for (int j = 0; j < 3; j++) {
        sg_pos[3 * t + j] = g.pos[j];
        sg_ls[3 * t + j] = g.ls[j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) sg_rot[4 * t + j] = g.rot[j];
    sg_logit[t] = g.logit;
#pragma unroll
    for (int j = 0; j < K3; j++) sg_sh[K3 * t + j] = g.sh[j];
}

template <int WIDTH>
__device__ __forceinline__ void adam_span(float *P, float *M, float *V, const float *sg,
                                          int64_t row0, int rows, float lr, const AdamF &c) {
    const int n = rows * WIDTH;
    float *p = P + WIDTH * row0, *m = M + WIDTH * row0, *v = V + WIDTH * row0;
    if (rows == 128) {
        // full CTA: 128 * WIDTH floats from WIDTH * row0 (row0 a multiple of
        // 128, so 16-byte aligned on 16-byte aligned arrays)
        for (int q = threadIdx.x; q < n / 4; q += 128) {
            float4 a = reinterpret_cast<float4 *>(p)[q];
            float4 b = reinterpret_cast<float4 *>(m)[q];
            float4 d = reinterpret_cast<float4 *>(v)[q];
            const float4 gg = reinterpret_cast<const float4 *>(sg)[q];
            adam_f32(a.x, b.x, d.x, gg.x, lr, c);
            adam_f32(a.y, b.y, d.y, gg.y, lr, c);
            adam_f32(a.z, b.z, d.z, gg.z, lr, c);
            adam_f32(a.w, b.w, d.w, gg.w, lr, c);
            reinterpret_cast<float4 *>(p)[q] = a;
            reinterpret_cast<float4 *>(m)[q] = b;
            reinterpret_cast<float4 *>(v)[q] = d;
        }
    } else {
        for (int q = threadIdx.x; q < n; q += 128) adam_f32(p[q], m[q], v[q], sg[q], lr, c);
    }
}

template <int K3, bool FOLD>
__global__ void __launch_bounds__(128, CFA_MINB) chain_fold_adam_f32_kernel(
    isg_train_state s, CamF cam, const uint8_t *__restrict__ flag,
    const double *__restrict__ grad2d, const int32_t *__restrict__ rank_of,
    const int64_t *__restrict__ live_off, const float4 *__restrict__ partials,
    const int4 *__restrict__ rect_sorted, int row_lo, int row_hi, int canon,
    double *__restrict__ grad2d_out, GradOut go, Lr5 lr, AdamF c, double half_w,
    double half_h) {
    __shared__ __align__(16) float sg_pos[3 * 128], sg_ls[3 * 128], sg_rot[4 * 128],
        sg_logit[128], sg_sh[K3 * 128];
    chain_rows_to_smem<K3, FOLD>(s, cam, flag, grad2d, rank_of, live_off, partials, rect_sorted,
                                 row_lo, row_hi, canon, grad2d_out, go, half_w, half_h, sg_pos,
                                 sg_ls, sg_rot, sg_logit, sg_sh);
    __syncthreads();
    const int64_t row0 = (int64_t)blockIdx.x * 128;
    const int rows = (int)min((int64_t)128, s.n - row0);
    adam_span<3>(s.positions, s.m_positions, s.v_positions, sg_pos, row0, rows, lr.v[0], c);
    adam_span<3>(s.log_scales, s.m_log_scales, s.v_log_scales, sg_ls, row0, rows, lr.v[1], c);
    adam_span<4>(s.rotations, s.m_rotations, s.v_rotations, sg_rot, row0, rows, lr.v[2], c);
    adam_span<1>(s.opacity_logits, s.m_opacity_logits, s.v_opacity_logits, sg_logit, row0, rows,
                 lr.v[3], c);
    adam_span<K3>(s.sh, s.m_sh, s.v_sh, sg_sh, row0, rows, lr.v[4], c);
}

void launch_chain_fold_adam_f32(const isg_train_state &st, const Cam &cam, const uint8_t *flag,
                                const double *grad2d, const int32_t *rank_of,
                                const int64_t *live_off, const float *partials,
                                const int32_t *rect_sorted, int row_lo, int row_hi, int canon,
                                double *grad2d_out, float *const *grads_out, const float *lr5,
                                const isg_adam_consts &ac, double half_w, double half_h,
                                cudaStream_t s) {
    const CamF c = to_camf(cam);
    const float4 *pt = reinterpret_cast<const float4 *>(partials);
    const int4 *rs = reinterpret_cast<const int4 *>(rect_sorted);
    GradOut go{nullptr, nullptr, nullptr, nullptr, nullptr};
    if (grads_out) go = GradOut{grads_out[0], grads_out[1], grads_out[2], grads_out[3], grads_out[4]};
    Lr5 lr;
    for (int k = 0; k < 5; k++) lr.v[k] = lr5[k];
    const AdamF a{(float)ac.b1, (float)ac.omb1, (float)ac.b2, (float)ac.omb2,
                  (float)ac.bc1, (float)ac.bc2, (float)ac.eps};
#define ISG_CFA(K, F)                                                                            \
    chain_fold_adam_f32_kernel<K, F><<<blocks_for(st.n, 128), 128, 0, s>>>(                      \
        st, c, flag, grad2d, rank_of, live_off, pt, rs, row_lo, row_hi, canon, grad2d_out, go, lr, \
        a, half_w, half_h)
    const bool fold = grad2d == nullptr;
    if (st.degree >= 1) {
        if (fold) ISG_CFA(12, true); else ISG_CFA(12, false);
    } else {
        if (fold) ISG_CFA(3, true); else ISG_CFA(3, false);
    }
#undef ISG_CFA
}

void launch_chain_fold_train_f32(const isg_params &p, const Cam &cam, const int32_t *rank_of,
                                 const int64_t *live_off, const float *partials,
                                 const int32_t *rect_sorted, int row_lo, int row_hi, int canon,
                                 double *grad2d_out, float *dpos, float *dls, float *drot,
                                 float *dlogit, float *dsh, int64_t *seen, double *grad_accum,
                                 double half_w, double half_h, cudaStream_t s) {
    const CamF c = to_camf(cam);
    const float4 *pt = reinterpret_cast<const float4 *>(partials);
    const int4 *rs = reinterpret_cast<const int4 *>(rect_sorted);
    if (p.degree >= 1)
        chain_fold_train_f32_kernel<12><<<blocks_for(p.n, 128), 128, 0, s>>>(
            p, c, rank_of, live_off, pt, rs, row_lo, row_hi, canon, grad2d_out, dpos, dls, drot,
            dlogit, dsh, seen, grad_accum, half_w, half_h);
    else
        chain_fold_train_f32_kernel<3><<<blocks_for(p.n, 128), 128, 0, s>>>(
            p, c, rank_of, live_off, pt, rs, row_lo, row_hi, canon, grad2d_out, dpos, dls, drot,
            dlogit, dsh, seen, grad_accum, half_w, half_h);
}

void launch_chain_train_f32(const isg_params &p, const Cam &cam, const uint8_t *flag,
                            const int32_t *rank_of, const double *grad2d, float *dpos,
                            float *dls, float *drot, float *dlogit, float *dsh, int64_t *seen,
                            double *grad_accum, double half_w, double half_h, cudaStream_t s) {
    const CamF c = to_camf(cam);
    if (p.degree >= 1)
        chain_train_f32_kernel<12><<<blocks_for(p.n, 128), 128, 0, s>>>(
            p, c, flag, rank_of, grad2d, dpos, dls, drot, dlogit, dsh, seen, grad_accum, half_w,
            half_h);
    else
        chain_train_f32_kernel<3><<<blocks_for(p.n, 128), 128, 0, s>>>(
            p, c, flag, rank_of, grad2d, dpos, dls, drot, dlogit, dsh, seen, grad_accum, half_w,
            half_h);
}

}  // namespace isg
