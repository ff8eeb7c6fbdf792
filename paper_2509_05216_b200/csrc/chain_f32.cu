// chain_f32.cu -- the training step's chain rule + TrainStats in float32
// (chain_f32.cuh), one thread per Gaussian row.  Rows find their 2-D
// gradients through rank_of (rank-ordered grad2d) or a visibility flag
// (row-ordered grad2d); stats are updated in float64 as in the reference
// (engine.py:508-515).  Built with FMA contraction (no bit-exact constraint).
#include "chain_f32.cuh"
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
