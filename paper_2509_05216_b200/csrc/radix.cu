// radix.cu -- hand-written stable LSD radix sort and exclusive scans (sm_100a).
//
// The sorts of the hot path (np.lexsort((indices, depth)) at
// rasterizer.py:161-163 / engine.py:213-215 and the tile regroup of
// build_tile_lists, rasterizer.py:166-191) and every prefix sum of the step.
// HBM-bound integer work, written for the B200 SM (no library code):
//
//   per 8-bit digit pass (reduce-then-scan, deterministic):
//     upsweep  : each CTA counts the digits of its 2048 keys (1024 for 64-bit
//                keys) in warp-private shared-memory counters -> counts[digit][cta]
//     scan     : digit-major exclusive scan of the counts (4096-element
//                chunks in shared memory + one CTA over the chunk sums)
//     scatter  : each warp loads its slice of the CTA's keys/values into
//                registers, ranks them stably (warp-level multi-split: peers
//                from one ballot per digit bit, per-warp digit counters,
//                warps in item order), permutes them into
//                digit order in shared memory and writes each digit run to
//                its global offset with consecutive threads on consecutive
//                addresses (coalesced stores)
//
// Stability: items are ranked in index order inside a CTA (warp w owns the
// w-th slice, lanes in order) and CTAs in index order through the scan, so
// each pass is stable and the LSD sequence sorts by the whole bit range.
#include <stdint.h>

#include "common.cuh"
#include "radix.cuh"

namespace isg {
namespace radix {

constexpr int RT = 256;        // threads per CTA
constexpr int NWARP = RT / 32;
// items per CTA (shared-memory staging: 64-bit keys take half as many)
#ifndef RADIX_IPC8
#define RADIX_IPC8 1024
#endif
#ifndef RADIX_IPC_SMALL
#define RADIX_IPC_SMALL 2048
#endif
template <typename K>
constexpr int ipc() { return sizeof(K) == 8 ? RADIX_IPC8 : RADIX_IPC_SMALL; }
constexpr int BINS = 256;
constexpr int SC = 4096;       // scan chunk (elements per CTA)


template <typename K>
__device__ __forceinline__ unsigned digit_of(K k, int shift, unsigned mask) {
    return (unsigned)((uint64_t)k >> shift) & mask;
}

// Lanes holding the same digit as this lane (warp-level multi-split by
// ballots over the digit bits; invalid lanes pass digit >= BINS, which no
// valid lane matches since bit 8 is compared too).
__device__ __forceinline__ unsigned digit_peers(unsigned d, int bits) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; b++) {
        if (b < bits || b == 8) {
            const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
    }
    return peers;
}

// Items per thread, and a thread's items as 16-byte vectors.
template <typename K>
constexpr int ipt() { return ipc<K>() / RT; }
template <typename K>
constexpr int kvec() { return ipt<K>() * (int)sizeof(K) / 16; }

template <typename K, bool VEC>
__global__ void __launch_bounds__(RT) upsweep_kernel(const K *__restrict__ keys, int64_t n,
                                                     int shift, unsigned mask, int nblk,
                                                     uint32_t *__restrict__ counts,
                                                     const int64_t *__restrict__ n_dev,
                                                     unsigned *__restrict__ done) {
    constexpr int IPC = ipc<K>(), IPT = ipt<K>();
    if (done && blockIdx.x == 0 && threadIdx.x == 0) *done = 0u;  // the scan's arrival counter
    if (n_dev) n = min(n, *n_dev);  // device-side item count (upper bound n)
    __shared__ uint32_t h[NWARP][BINS];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < NWARP * BINS; i += RT) (&h[0][0])[i] = 0u;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * IPC;
    const int nv = (int)max((int64_t)0, min((int64_t)IPC, n - base));
    if (VEC && nv == IPC) {
        // blocked: thread t owns items [t * IPT, (t + 1) * IPT), all loads in flight
        union {
            uint4 v[kvec<K>()];
            K k[IPT];
        } u;
        const uint4 *src = reinterpret_cast<const uint4 *>(keys + base) + threadIdx.x * kvec<K>();
#pragma unroll
        for (int q = 0; q < kvec<K>(); q++) u.v[q] = __ldg(src + q);
#pragma unroll
        for (int q = 0; q < IPT; q++) atomicAdd(&h[warp][digit_of(u.k[q], shift, mask)], 1u);
    } else {
        for (int i = threadIdx.x; i < nv; i += RT)
            atomicAdd(&h[warp][digit_of(keys[base + i], shift, mask)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += RT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < NWARP; w++) s += h[w][d];
        counts[(int64_t)d * nblk + blockIdx.x] = s;
    }
}

// Exclusive scan of a CTA's chunk of SC elements (in -> out, may alias);
// chunk total to sums.  Coalesced through shared memory.
template <typename T>
__global__ void __launch_bounds__(RT) scan_chunks_kernel(const T *in, T *out, int64_t n,
                                                         T *__restrict__ sums,
                                                         unsigned *__restrict__ done) {
    constexpr int PER = SC / RT;  // elements per thread (contiguous in shared memory)
    // one pad element per PER: thread t's run starts t * (PER + 1) elements in,
    // so a warp's lanes read different banks (unpadded, every lane of the
    // warp hit the same bank at each step)
    __shared__ T sm[SC + SC / PER];
    __shared__ T swarp[NWARP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cb = (int64_t)blockIdx.x * SC;
    auto at = [](int i) { return i + i / PER; };
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int64_t i = cb + k * RT + threadIdx.x;
        sm[at(k * RT + threadIdx.x)] = i < n ? in[i] : (T)0;
    }
    __syncthreads();
    T v[PER];
    T s = 0;
#pragma unroll
    for (int k = 0; k < PER; k++) {
        v[k] = sm[at(threadIdx.x * PER + k)];
        s += v[k];
    }
    T x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) swarp[warp] = x;
    __syncthreads();
    T before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < NWARP; w++) {
        if (w < warp) before += swarp[w];
        total += swarp[w];
    }
    T run = before + x - s;
#pragma unroll
    for (int k = 0; k < PER; k++) {
        sm[at(threadIdx.x * PER + k)] = run;
        run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int64_t i = cb + k * RT + threadIdx.x;
        if (i < n) out[i] = sm[at(k * RT + threadIdx.x)];
    }
    // the last CTA to finish scans the chunk sums in place (no separate
    // launch); done: an arrival counter that starts at 0 and is left at 0
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        sums[blockIdx.x] = total;
        if (done) {
            __threadfence();
            s_last = atomicAdd(done, 1u) == gridDim.x - 1;
        }
    }
    if (!done) return;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int m = (int)gridDim.x;
    T carry = 0;
    for (int c0 = 0; c0 < m; c0 += RT) {
        const int i = c0 + threadIdx.x;
        const T v = i < m ? reinterpret_cast<volatile T *>(sums)[i] : (T)0;
        T y = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        if (lane == 31) swarp[warp] = y;
        __syncthreads();
        T pre = carry, tot = 0;
#pragma unroll
        for (int w = 0; w < NWARP; w++) {
            if (w < warp) pre += swarp[w];
            tot += swarp[w];
        }
        if (i < m) sums[i] = pre + y - v;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *done = 0u;
}

template <typename K, bool VEC>
__global__ void __launch_bounds__(RT) scatter_kernel(const K *__restrict__ keys_in,
                                                     const int32_t *__restrict__ vals_in,
                                                     K *__restrict__ keys_out,
                                                     int32_t *__restrict__ vals_out, int64_t n,
                                                     int shift, unsigned mask, int nblk,
                                                     const uint32_t *__restrict__ offs,
                                                     const uint32_t *__restrict__ chunk_off,
                                                     const int64_t *__restrict__ n_dev) {
    constexpr int IPC = ipc<K>(), IPT = ipt<K>();
    constexpr int SLICE = IPC / NWARP;  // = 32 * IPT
    const int bits = __popc(mask);
    extern __shared__ __align__(16) unsigned char smem[];
    K *sk = reinterpret_cast<K *>(smem);                   // digit-ordered staging
    int32_t *sv = reinterpret_cast<int32_t *>(sk + IPC);
    __shared__ uint32_t wcnt[NWARP][BINS];
    __shared__ uint32_t dstart[BINS];
    __shared__ int64_t gdelta[BINS];
    __shared__ uint32_t sw[NWARP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (n_dev) n = min(n, *n_dev);
    const int64_t base = (int64_t)blockIdx.x * IPC;
    if (base >= n) return;
    const int nv = (int)min((int64_t)IPC, n - base);
    for (int i = threadIdx.x; i < NWARP * BINS; i += RT) (&wcnt[0][0])[i] = 0u;
    // a warp's slice, lane-interleaved: item r * 32 + lane of the slice
    K k[IPT];
    int32_t v[IPT];
    const int64_t sbase = base + warp * SLICE;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int i = warp * SLICE + r * 32 + lane;
        if (i < nv) {
            k[r] = keys_in[sbase + r * 32 + lane];
            v[r] = vals_in[sbase + r * 32 + lane];
        }
    }
    __syncthreads();
    // warp-level multi-split: rank of every item among the same digit in its
    // slice (items in slice order), kept in registers
    uint32_t lp[IPT];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const bool valid = warp * SLICE + r * 32 + lane < nv;
        const unsigned d = valid ? digit_of(k[r], shift, mask) : BINS;
        const unsigned peers = digit_peers(d, bits);
        uint32_t c = 0;
        if (valid) c = wcnt[warp][d];
        lp[r] = c + __popc(peers & lt);
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) wcnt[warp][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: warp prefixes, CTA total; exclusive scan over digits
    const int d = threadIdx.x;  // RT == BINS
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < NWARP; w++) {
        const uint32_t c = wcnt[w][d];
        wcnt[w][d] = tot;
        tot += c;
    }
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    const int64_t ci = (int64_t)d * nblk + blockIdx.x;
    const int64_t go = (int64_t)offs[ci] + chunk_off[ci / SC];
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < NWARP; w++)
        if (w < warp) before += sw[w];
    const uint32_t ds = before + x - tot;
    dstart[d] = ds;
    gdelta[d] = go - (int64_t)ds;
    __syncthreads();
    // permute into digit order in shared memory
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        if (warp * SLICE + r * 32 + lane < nv) {
            const unsigned dd = digit_of(k[r], shift, mask);
            const uint32_t dest = dstart[dd] + wcnt[warp][dd] + lp[r];
            sk[dest] = k[r];
            sv[dest] = v[r];
        }
    }
    __syncthreads();
    // each digit run to its global offset (consecutive threads, consecutive addresses)
    for (int j = threadIdx.x; j < nv; j += RT) {
        const K kk = sk[j];
        const int64_t g = gdelta[digit_of(kk, shift, mask)] + j;
        keys_out[g] = kk;
        vals_out[g] = sv[j];
    }
}

// 2- and 4-byte keys: the CTA's items staged in shared memory with 16-byte
// vector loads, ranked, permuted into a second staging area, written out.
template <typename K, bool VEC>
__global__ void __launch_bounds__(RT) scatter_staged_kernel(const K *__restrict__ keys_in,
                                                     const int32_t *__restrict__ vals_in,
                                                     K *__restrict__ keys_out,
                                                     int32_t *__restrict__ vals_out, int64_t n,
                                                     int shift, unsigned mask, int nblk,
                                                     const uint32_t *__restrict__ offs,
                                                     const uint32_t *__restrict__ chunk_off,
                                                     const int64_t *__restrict__ n_dev) {
    constexpr int IPC = ipc<K>();
    constexpr int SLICE = IPC / NWARP;
    const int bits = __popc(mask);
    extern __shared__ __align__(16) unsigned char smem[];
    K *sk = reinterpret_cast<K *>(smem);
    K *sk2 = sk + IPC;
    int32_t *sv = reinterpret_cast<int32_t *>(sk2 + IPC);
    int32_t *sv2 = sv + IPC;
    uint16_t *slp = reinterpret_cast<uint16_t *>(sv2 + IPC);
    __shared__ uint32_t wcnt[NWARP][BINS];
    __shared__ uint32_t dstart[BINS];
    __shared__ uint32_t goff[BINS];
    __shared__ uint32_t sw[NWARP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (n_dev) n = min(n, *n_dev);
    const int64_t base = (int64_t)blockIdx.x * IPC;
    if (base >= n) return;
    const int nv = (int)min((int64_t)IPC, n - base);
    if (VEC && nv == IPC) {
        // all of a thread's loads in flight at once (16-byte vectors), then
        // staged in shared memory at the same positions
        constexpr int KV = kvec<K>(), VV = ipt<K>() / 4;
        uint4 kv[KV], vv[VV];
        const uint4 *ks = reinterpret_cast<const uint4 *>(keys_in + base) + threadIdx.x * KV;
        const uint4 *vs = reinterpret_cast<const uint4 *>(vals_in + base) + threadIdx.x * VV;
#pragma unroll
        for (int q = 0; q < KV; q++) kv[q] = __ldg(ks + q);
#pragma unroll
        for (int q = 0; q < VV; q++) vv[q] = __ldg(vs + q);
#pragma unroll
        for (int q = 0; q < KV; q++) reinterpret_cast<uint4 *>(sk)[threadIdx.x * KV + q] = kv[q];
#pragma unroll
        for (int q = 0; q < VV; q++) reinterpret_cast<uint4 *>(sv)[threadIdx.x * VV + q] = vv[q];
    } else {
        for (int i = threadIdx.x; i < nv; i += RT) {
            sk[i] = keys_in[base + i];
            sv[i] = vals_in[base + i];
        }
    }
    for (int i = threadIdx.x; i < NWARP * BINS; i += RT) (&wcnt[0][0])[i] = 0u;
    __syncthreads();
    // warp-level multi-split: local rank of every item among the same digit
    // in its warp slice (slices in warp order = item order)
    for (int i = warp * SLICE + lane; i < (warp + 1) * SLICE; i += 32) {
        const bool valid = i < nv;
        const unsigned d = valid ? digit_of(sk[i], shift, mask) : BINS;
        const unsigned peers = digit_peers(d, bits);
        const unsigned lt = (1u << lane) - 1u;
        uint32_t lp = 0;
        if (valid) lp = wcnt[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) wcnt[warp][d] += __popc(peers);
        __syncwarp();
        if (valid) slp[i] = (uint16_t)lp;
    }
    __syncthreads();
    // per digit: warp prefixes, CTA total; exclusive scan over digits
    const int d = threadIdx.x;  // RT == BINS
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < NWARP; w++) {
        const uint32_t c = wcnt[w][d];
        wcnt[w][d] = tot;
        tot += c;
    }
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    const int64_t ci = (int64_t)d * nblk + blockIdx.x;
    goff[d] = offs[ci] + chunk_off[ci / SC];
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < NWARP; w++)
        if (w < warp) before += sw[w];
    dstart[d] = before + x - tot;
    __syncthreads();
    // permute into digit order in shared memory
    for (int i = threadIdx.x; i < nv; i += RT) {
        const unsigned dd = digit_of(sk[i], shift, mask);
        const uint32_t dest = dstart[dd] + wcnt[i / SLICE][dd] + slp[i];
        sk2[dest] = sk[i];
        sv2[dest] = sv[i];
    }
    __syncthreads();
    // each digit run to its global offset (consecutive threads, consecutive addresses)
    for (int j = threadIdx.x; j < nv; j += RT) {
        const K k = sk2[j];
        const unsigned dd = digit_of(k, shift, mask);
        const int64_t g = (int64_t)goff[dd] + (j - (int64_t)dstart[dd]);
        keys_out[g] = k;
        vals_out[g] = sv2[j];
    }
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// 8-byte keys: items in registers (scatter_kernel); smaller keys: staged
// twice in shared memory (scatter_staged_kernel)
template <typename K>
constexpr bool staged() { return sizeof(K) < 8; }
template <typename K>
constexpr size_t scatter_smem() {
    return staged<K>() ? (size_t)ipc<K>() * (2 * (sizeof(K) + sizeof(int32_t)) + sizeof(uint16_t))
                       : (size_t)ipc<K>() * (sizeof(K) + sizeof(int32_t));
}

// Workspace: key/value ping-pong buffers, digit counts, chunk sums.
template <typename K>
size_t sort_ws_bytes(int64_t n) {
    const int64_t nblk = (n + ipc<K>() - 1) / ipc<K>();
    const int64_t nc = (int64_t)BINS * nblk;
    const int64_t nch = (nc + SC - 1) / SC;
    return al(sizeof(K) * (size_t)n) + al(sizeof(int32_t) * (size_t)n) +
           al(sizeof(uint32_t) * (size_t)nc) + al(sizeof(uint32_t) * (size_t)(nch + 1)) +
           al(sizeof(unsigned));
}

template <typename K>
int sort_pairs(void *ws, size_t *ws_bytes, const K *keys_in, K *keys_out,
               const int32_t *vals_in, int32_t *vals_out, int64_t n, int b0, int b1,
               cudaStream_t s, const int64_t *n_dev) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || b0 < 0 || b1 > (int)(8 * sizeof(K)) || b0 >= b1)
        return (int)cudaErrorInvalidValue;
    const size_t need = sort_ws_bytes<K>(n);
    if (!ws) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    const int64_t nblk = (n + ipc<K>() - 1) / ipc<K>();
    const int64_t nc = (int64_t)BINS * nblk;
    const int64_t nch = (nc + SC - 1) / SC;
    char *p = (char *)ws;
    K *k_alt = (K *)p;
    p += al(sizeof(K) * (size_t)n);
    int32_t *v_alt = (int32_t *)p;
    p += al(sizeof(int32_t) * (size_t)n);
    uint32_t *counts = (uint32_t *)p;
    p += al(sizeof(uint32_t) * (size_t)nc);
    uint32_t *csum = (uint32_t *)p;
    p += al(sizeof(uint32_t) * (size_t)(nch + 1));
    unsigned *done = (unsigned *)p;  // zeroed by the first upsweep CTA each pass
    const int passes = (b1 - b0 + 7) / 8;
    for (auto fn : {scatter_kernel<K, true>, scatter_kernel<K, false>,
                    scatter_staged_kernel<K, true>, scatter_staged_kernel<K, false>}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)scatter_smem<K>());
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return (int)e;
    }
    // ping-pong so that the last pass writes keys_out / vals_out
    const K *src_k = keys_in;
    const int32_t *src_v = vals_in;
    for (int q = 0; q < passes; q++) {
        const int shift = b0 + 8 * q;
        const int bits = min(8, b1 - shift);
        const unsigned mask = (1u << bits) - 1u;
        const bool to_out = ((passes - 1 - q) & 1) == 0;
        K *dst_k = to_out ? keys_out : k_alt;
        int32_t *dst_v = to_out ? vals_out : v_alt;
        // 16-byte vector loads when every array of this pass is aligned
        const bool vec = ((uintptr_t)src_k % 16 == 0) && ((uintptr_t)src_v % 16 == 0);
        if (vec)
            upsweep_kernel<K, true><<<(unsigned)nblk, RT, 0, s>>>(src_k, n, shift, mask,
                                                                  (int)nblk, counts, n_dev, done);
        else
            upsweep_kernel<K, false><<<(unsigned)nblk, RT, 0, s>>>(src_k, n, shift, mask,
                                                                   (int)nblk, counts, n_dev, done);
        ISG_CHECK_LAUNCH();
        scan_chunks_kernel<uint32_t><<<(unsigned)nch, RT, 0, s>>>(counts, counts, nc, csum, done);
        ISG_CHECK_LAUNCH();
        if (!staged<K>())
            scatter_kernel<K, true><<<(unsigned)nblk, RT, scatter_smem<K>(), s>>>(
                src_k, src_v, dst_k, dst_v, n, shift, mask, (int)nblk, counts, csum, n_dev);
        else if (vec)
            scatter_staged_kernel<K, true><<<(unsigned)nblk, RT, scatter_smem<K>(), s>>>(
                src_k, src_v, dst_k, dst_v, n, shift, mask, (int)nblk, counts, csum, n_dev);
        else
            scatter_staged_kernel<K, false><<<(unsigned)nblk, RT, scatter_smem<K>(), s>>>(
                src_k, src_v, dst_k, dst_v, n, shift, mask, (int)nblk, counts, csum, n_dev);
        ISG_CHECK_LAUNCH();
        src_k = dst_k;
        src_v = dst_v;
    }
    return 0;
}

}  // namespace radix

// Exclusive int64 scan: off[0] = 0, off[i + 1] = cnt[0] + ... + cnt[i]; total
// (device, optional) = off[n].  Workspace: the chunk sums.
size_t scan_i64_ws_bytes(int64_t n) {
    return radix::al(sizeof(int64_t) * (size_t)((n + radix::SC - 1) / radix::SC + 1)) +
           radix::al(sizeof(unsigned));
}


__global__ void scan_tail_kernel(int64_t n, int64_t *__restrict__ off,
                                 const int64_t *__restrict__ csum, const int64_t *__restrict__ cnt,
                                 int64_t *__restrict__ total) {
    // off[0..n) holds chunk-local exclusive prefixes of cnt; add chunk offsets
    // and append the total
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) off[i] += csum[i / radix::SC];
    if (i == n - 1) {
        const int64_t t = off[i] + cnt[i];
        off[n] = t;
        if (total) *total = t;
    }
}

int scan_i64(void *ws, size_t ws_bytes, int64_t n, const int64_t *cnt, int64_t *off,
             int64_t *total, cudaStream_t s) {
    if (n < 0 || ws_bytes < scan_i64_ws_bytes(n)) return (int)cudaErrorInvalidValue;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(off, 0, sizeof(int64_t), s);
        if (e == cudaSuccess && total) e = cudaMemsetAsync(total, 0, sizeof(int64_t), s);
        return (int)e;
    }
    const int64_t nch = (n + radix::SC - 1) / radix::SC;
    int64_t *csum = (int64_t *)ws;
    unsigned *done = (unsigned *)((char *)ws + radix::al(sizeof(int64_t) * (size_t)(nch + 1)));
    cudaError_t e = cudaMemsetAsync(done, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return (int)e;
    radix::scan_chunks_kernel<int64_t><<<(unsigned)nch, radix::RT, 0, s>>>(cnt, off, n, csum,
                                                                            done);
    ISG_CHECK_LAUNCH();
    scan_tail_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, off, csum, cnt, total);
    ISG_CHECK_LAUNCH();
    return 0;
}

template int radix::sort_pairs<uint16_t>(void *, size_t *, const uint16_t *, uint16_t *,
                                         const int32_t *, int32_t *, int64_t, int, int,
                                         cudaStream_t, const int64_t *);
template int radix::sort_pairs<uint32_t>(void *, size_t *, const uint32_t *, uint32_t *,
                                         const int32_t *, int32_t *, int64_t, int, int,
                                         cudaStream_t, const int64_t *);
template int radix::sort_pairs<uint64_t>(void *, size_t *, const uint64_t *, uint64_t *,
                                         const int32_t *, int32_t *, int64_t, int, int,
                                         cudaStream_t, const int64_t *);

}  // namespace isg
