// adam.cuh -- the float32 Adam update shared by every launch that applies it.
#pragma once

namespace isg {

struct AdamF {
    float b1, omb1, b2, omb2, bc1, bc2, eps;
};

// optim.py:49-55 in float32 with numpy's operation order: every operation
// rounded on its own (explicit _rn intrinsics, so no translation unit's FMA
// contraction setting can change the bits).
__device__ __forceinline__ void adam_f32(float &p, float &m, float &v, float g, float lr,
                                         const AdamF &c) {
    const float mi = __fadd_rn(__fmul_rn(m, c.b1), __fmul_rn(c.omb1, g));
    const float vi = __fadd_rn(__fmul_rn(v, c.b2), __fmul_rn(c.omb2, __fmul_rn(g, g)));
    const float mhat = __fdiv_rn(mi, c.bc1);
    const float vhat = __fdiv_rn(vi, c.bc2);
    const float den = __fadd_rn(__fsqrt_rn(vhat), c.eps);
    const float step = __fdiv_rn(__fmul_rn(lr, mhat), den);
    p = __fsub_rn(p, step);
    m = mi;
    v = vi;
}

}  // namespace isg
