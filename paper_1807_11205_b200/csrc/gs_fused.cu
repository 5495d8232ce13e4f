// gs_fused.cu — collective + LARS pass fused into single kernels over NVLink
// peer memory (the sharded, ZeRO-1 form of the step).
//
//   gs_rs_pass1   reduce-scatter fused with pass 1: the owner of a chunk reads
//                 every peer's raw binary16 values of that chunk over NVLink,
//                 folds them in the reference's pairwise-tree order
//                 (fold_f16_tree, collectives.py:273-283), stores the reduced
//                 chunk in its own wire and immediately runs pass 1 on the
//                 folded registers (no re-read), then PUSHES the chunk's fp64
//                 partials to every peer and ORs its flags into every peer's
//                 flag word (remote stores / atomics) — no gather kernel.
//   gs_pass2_push pass 2 over the owned chunks that also pushes each updated
//                 binary16 working-weight vector to every peer's working
//                 arena — no all-gather kernel.
//   gs_peer_fence one CTA: every rank has finished the previous kernels'
//                 remote stores (system fence + release/acquire signals).
// The per-chunk arithmetic (p1_vec / p2_pair / block_sum3, thread-to-element
// mapping, fold order) is exactly the LARS kernels', so the partials, trust
// scales and updates are bit-identical to the replicated path.
#include "gs_lars_device.cuh"
#include "gs_peer.cuh"

namespace {

// vectors per thread in flight per batch (P raw loads each).  One vector
// keeps the kernel at <= 64 registers for P = 2 / 4 (4 co-resident CTAs per
// SM) and <= 80 for P = 8 (3 per SM): the reduce-scatter is bound by NVLink
// load latency per chunk, so more resident CTAs = more chunks in flight
// (two vectors took 124-206 registers, 1-2 CTAs per SM)
template <int P>
constexpr int kU = 1;

template <int P, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY>
__device__ __forceinline__ void rs_p1_chunk(const uint16_t* const (&src)[P], uint16_t* mine,
                                            const float* __restrict__ w, int len, const Ctx& cx,
                                            Acc& a) {
  bool vec = gs::is_aligned16(mine) && (!LARS || gs::is_aligned16(w));
#pragma unroll
  for (int q = 0; q < P; ++q) vec = vec && gs::is_aligned16(src[q]);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // vectors t, t+256, ... in increasing order: the summation order of pass 1
  for (int base = t; base < nv; base += kU<P> * kThreads) {
    uint4 raw[kU<P>][P];
    F8 wv[kU<P>];
#pragma unroll
    for (int u = 0; u < kU<P>; ++u) {
      const int i = base + u * kThreads;
      if (i < nv) {
#pragma unroll
        for (int q = 0; q < P; ++q) raw[u][q] = __ldcv(reinterpret_cast<const uint4*>(src[q]) + i);
        if (LARS) wv[u] = ldw(w + 8 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU<P>; ++u) {
      const int i = base + u * kThreads;
      if (i >= nv) break;
      uint4 o;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float x[P], y[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const float2 f = gs::widen2((&raw[u][q].x)[h]);
          x[q] = f.x;
          y[q] = f.y;
        }
        (&o.x)[h] = gs::narrow2(tree<P>(x), tree<P>(y));
      }
      reinterpret_cast<uint4*>(mine)[i] = o;
      p1_vec<true, POW2, RAWFLAG, GNORM, LARS, DECAY>(o, LARS ? wv[u] : F8{}, cx, a);
    }
  }
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = gs::widen(__ldcv(src[q] + i));
    const uint16_t h = gs::narrow(tree<P>(v));
    mine[i] = h;
    if (RAWFLAG) a.raw |= raw_nonfinite_bits(h);
    Acc b;
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY>(make_float2(gs::widen(h), 0.0f),
                                               make_float2(LARS ? w[i] : 0.0f, 0.0f), cx, b);
    a.sw += b.sw;
    a.se += b.se;
    a.sg += b.sg;
    a.fl |= b.fl;
  }
}

// cp.async (LDGSTS) 16-byte copy global -> shared, L2 only (peer addresses are
// plain global addresses mapped over NVLink)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// vectors of a full chunk per thread (8192 / 256 / 8)
constexpr int kChunkIters = kFullChunk / (kThreads * 8);

// shared-memory staging of one chunk: [iter][source q = 0..P-1, w lo, w hi][thread]
template <int P>
constexpr int kStageBytes = kChunkIters * (P + 2) * kThreads * 16;

// The staged form of rs_p1_chunk: every thread issues ALL its vectors' peer
// loads (and master loads) for the chunk as cp.async copies into its own
// shared-memory slots at once, waits for its own copies only (no CTA
// barrier: a thread reads back nothing but what it staged), then folds and
// runs pass 1 in the same per-thread vector order as rs_p1_chunk — so the
// results are bit-identical; only the memory-level parallelism changes
// (P x 4 x 16 B per thread in flight instead of P x 16 B).
template <int P, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY>
__device__ __forceinline__ void rs_p1_chunk_staged(const uint16_t* const (&src)[P], uint16_t* mine,
                                                   const float* __restrict__ w, int len,
                                                   const Ctx& cx, Acc& a, uint4* stage) {
  bool vec = gs::is_aligned16(mine) && (!LARS || gs::is_aligned16(w)) && len <= kFullChunk;
#pragma unroll
  for (int q = 0; q < P; ++q) vec = vec && gs::is_aligned16(src[q]);
  if (!vec) {
    rs_p1_chunk<P, POW2, RAWFLAG, GNORM, LARS, DECAY>(src, mine, w, len, cx, a);
    return;
  }
  const int nv = len / 8;
  const int t = threadIdx.x;
  auto slot = [&](int it, int q) -> uint4* { return stage + (it * (P + 2) + q) * kThreads + t; };
#pragma unroll
  for (int it = 0; it < kChunkIters; ++it) {
    const int i = t + it * kThreads;
    if (i < nv) {
#pragma unroll
      for (int q = 0; q < P; ++q) cp_async16(slot(it, q), reinterpret_cast<const uint4*>(src[q]) + i);
      if (LARS) {
        cp_async16(slot(it, P), reinterpret_cast<const uint4*>(w + 8 * i));
        cp_async16(slot(it, P + 1), reinterpret_cast<const uint4*>(w + 8 * i) + 1);
      }
    }
  }
  cp_async_wait_all();
#pragma unroll 1
  for (int it = 0; it < kChunkIters; ++it) {
    const int i = t + it * kThreads;
    if (i >= nv) break;
    uint4 o;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float x[P], y[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const float2 f = gs::widen2((&slot(it, q)->x)[h]);
        x[q] = f.x;
        y[q] = f.y;
      }
      (&o.x)[h] = gs::narrow2(tree<P>(x), tree<P>(y));
    }
    reinterpret_cast<uint4*>(mine)[i] = o;
    F8 wv{};
    if (LARS) {
      const uint4 lo = *slot(it, P), hi = *slot(it, P + 1);
      wv.a = make_float4(__uint_as_float(lo.x), __uint_as_float(lo.y), __uint_as_float(lo.z),
                         __uint_as_float(lo.w));
      wv.b = make_float4(__uint_as_float(hi.x), __uint_as_float(hi.y), __uint_as_float(hi.z),
                         __uint_as_float(hi.w));
    }
    p1_vec<true, POW2, RAWFLAG, GNORM, LARS, DECAY>(o, wv, cx, a);
  }
  // scalar tail (len not a multiple of 8): the direct path's loop
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = gs::widen(__ldcv(src[q] + i));
    const uint16_t h = gs::narrow(tree<P>(v));
    mine[i] = h;
    if (RAWFLAG) a.raw |= raw_nonfinite_bits(h);
    Acc b;
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY>(make_float2(gs::widen(h), 0.0f),
                                               make_float2(LARS ? w[i] : 0.0f, 0.0f), cx, b);
    a.sw += b.sw;
    a.se += b.se;
    a.sg += b.sg;
    a.fl |= b.fl;
  }
}

// residency: every CTA waits for its peers at entry, so the whole grid must
// fit at once (the launcher clamps the grid with the occupancy calculator)
template <int P>
constexpr int kRsMinBlocks = P <= 4 ? 4 : 3;

template <int P, bool POW2, bool RAWFLAG, bool GNORM, bool STAGE>
__global__ void __launch_bounds__(kThreads, kRsMinBlocks<P>)
rs_pass1_kernel(const uint64_t* __restrict__ wires, const uint8_t* own_wire,
                const uint64_t* __restrict__ sig, int rank, const gs_segment* __restrict__ segs, const gs_chunk* __restrict__ chunks, int c0,
                int c1, const int32_t* __restrict__ chunk_list, const gs_step_params* __restrict__ params,
                const uint64_t* __restrict__ peer_partials, const uint64_t* __restrict__ peer_flags,
                uint32_t epoch, const uint32_t* __restrict__ epoch_base) {
  epoch += *epoch_base;
  // every rank's bucket is packed (pull form: into its own wire; inbox form:
  // stored into the owners' inboxes over NVLink) -- a release signal,
  // cumulative over those stream-ordered stores
  peer_barrier(sig, rank, P, 0, epoch);
  Ctx cx;
  cx.u.load(params);
  cx.mul = params->mul;
  cx.wd = params->weight_decay;
  // src[q] = wires[q] + (chunk's byte offset in my wire)
  const uint8_t* mybase =
      own_wire != nullptr ? own_wire : reinterpret_cast<const uint8_t*>(wires[rank]);
  uint32_t flag_acc = 0;
  for (int ci = c0 + blockIdx.x; ci < c1; ci += gridDim.x) {
    const int c = chunk_list != nullptr ? chunk_list[ci] : ci;
    const gs_chunk ch = chunks[c];
    const gs_segment* sp = segs + ch.seg;
    const uint32_t sflags = sp->flags;
    uint16_t* mine = const_cast<uint16_t*>(static_cast<const uint16_t*>(sp->g)) + ch.start;
    const size_t off = reinterpret_cast<const uint8_t*>(mine) - mybase;
    const uint16_t* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const uint16_t*>(wires[q] + off);
    const float* w = sp->w + ch.start;
    const bool lars = (sflags & GS_SEG_LARS_ENABLED) != 0;
    const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
    Acc a;
    if (STAGE) {
      extern __shared__ uint4 stage[];
      if (lars && decay)
        rs_p1_chunk_staged<P, POW2, RAWFLAG, GNORM, true, true>(src, mine, w, ch.len, cx, a, stage);
      else if (lars)
        rs_p1_chunk_staged<P, POW2, RAWFLAG, GNORM, true, false>(src, mine, w, ch.len, cx, a, stage);
      else
        rs_p1_chunk_staged<P, POW2, RAWFLAG, GNORM, false, false>(src, mine, w, ch.len, cx, a, stage);
    } else if (lars && decay) {
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, true, true>(src, mine, w, ch.len, cx, a);
    } else if (lars) {
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, true, false>(src, mine, w, ch.len, cx, a);
    } else {
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, false, false>(src, mine, w, ch.len, cx, a);
    }
    if (lars && !decay) {
      a.se = a.sg;
      if (!GNORM) a.sg = 0.0;
    }
    flag_acc |= a.fl | ((a.raw & 0x80008000u) ? kBoth : 0u);
    double sw = a.sw, se = a.se, sg = a.sg;
    gs::block_sum3<kThreads>(sw, se, sg);
    // push the chunk partial into every rank's partials (own included)
    __shared__ double s_part[3];
    if (threadIdx.x == 0) {
      s_part[0] = sw;
      s_part[1] = se;
      s_part[2] = sg;
    }
    __syncthreads();
    if (threadIdx.x < P) {
      double* dst = reinterpret_cast<double*>(peer_partials[threadIdx.x]) + 3 * (int64_t)c;
      dst[0] = s_part[0];
      dst[1] = s_part[1];
      dst[2] = s_part[2];
    }
    __syncthreads();  // block_sum3 scratch and s_part are reused next chunk
  }
  flag_acc = __reduce_or_sync(0xFFFFFFFFu, flag_acc);
  if (flag_acc != 0u && (threadIdx.x & 31) == 0) {
    for (int q = 0; q < P; ++q)
      atomicOr_system(reinterpret_cast<unsigned int*>(peer_flags[q]), flag_acc);
  }
}

// NVLS multicast store: ONE 16-byte store to a multicast address that the
// NVSwitch replicates into every rank's copy (the bits travel untouched)
__device__ __forceinline__ void multimem_st16(uint8_t* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc),
               "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
               "f"(__uint_as_float(v.w))
               : "memory");
}

// pass 2 over owned chunks, pushing the binary16 result to every peer: with
// a multicast mapping of the working arena (mc != nullptr) one multimem
// store per vector reaches every rank (outbound NVLink traffic 1x instead of
// (p-1)x); otherwise one store per peer
template <bool POW2, bool DECAY>
__device__ __forceinline__ void p2_push_chunk(const uint16_t* __restrict__ g, float* __restrict__ w,
                                              float* __restrict__ v, uint16_t* __restrict__ w16,
                                              int len, const Ctx& cx, float s,
                                              const uint64_t* __restrict__ peer_working, int p,
                                              int rank, size_t woff, uint8_t* mc) {
  using Gt = G<true>;
  const bool vec = gs::is_aligned16(g) && gs::is_aligned16(w) && gs::is_aligned16(v) &&
                   gs::is_aligned16(w16);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // one 8-element vector: update in registers, local v/w streaming stores,
  // binary16 result stored into every rank's working arena (own included)
  auto one = [&](const uint4& gv, const F8& wv, const F8& vv, int i) {
    float2 ww[4] = {make_float2(wv.a.x, wv.a.y), make_float2(wv.a.z, wv.a.w),
                    make_float2(wv.b.x, wv.b.y), make_float2(wv.b.z, wv.b.w)};
    float2 xv[4] = {make_float2(vv.a.x, vv.a.y), make_float2(vv.a.z, vv.a.w),
                    make_float2(vv.b.x, vv.b.y), make_float2(vv.b.z, vv.b.w)};
#pragma unroll
    for (int q = 0; q < 4; ++q) p2_pair<POW2, DECAY>(Gt::pair(gv, q), ww[q], xv[q], cx, s);
    float4* vp = reinterpret_cast<float4*>(v) + 2 * i;
    float4* wp = reinterpret_cast<float4*>(w) + 2 * i;
    __stcs(vp, make_float4(xv[0].x, xv[0].y, xv[1].x, xv[1].y));
    __stcs(vp + 1, make_float4(xv[2].x, xv[2].y, xv[3].x, xv[3].y));
    __stcs(wp, make_float4(ww[0].x, ww[0].y, ww[1].x, ww[1].y));
    __stcs(wp + 1, make_float4(ww[2].x, ww[2].y, ww[3].x, ww[3].y));
    const uint4 h = make_uint4(pack_w16(ww[0]), pack_w16(ww[1]), pack_w16(ww[2]), pack_w16(ww[3]));
    if (mc != nullptr) {
      multimem_st16(mc + woff + 16 * (size_t)i, h);
    } else {
      for (int q = 0; q < p; ++q)
        reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(peer_working[q]) + woff)[i] = h;
    }
  };
  // batches of two vectors per thread with every load issued first (the
  // stores cannot alias the next batch's loads, which the compiler cannot
  // prove through the casts) -- the same batching as lars_pass2
  int done = 0;
  for (; done + 2 * kThreads <= nv; done += 2 * kThreads) {
    const int i0 = done + t, i1 = i0 + kThreads;
    const uint4 g0 = Gt::ld(g + 8 * i0), g1 = Gt::ld(g + 8 * i1);
    const F8 w0 = ld8(w, i0), w1 = ld8(w, i1), v0 = ld8(v, i0), v1 = ld8(v, i1);
    one(g0, w0, v0, i0);
    one(g1, w1, v1, i1);
  }
  for (int i = done + t; i < nv; i += kThreads) one(Gt::ld(g + 8 * i), ld8(w, i), ld8(v, i), i);
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float2 ww = make_float2(w[i], 0.0f), vv = make_float2(v[i], 0.0f);
    p2_pair<POW2, DECAY>(make_float2(Gt::one(g + i), 0.0f), ww, vv, cx, s);
    v[i] = vv.x;
    w[i] = ww.x;
    const uint16_t h = gs::narrow(ww.x);
    for (int q = 0; q < p; ++q)
      reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(peer_working[q]) + woff)[i] = h;
  }
}

template <bool POW2>
__global__ void __launch_bounds__(kThreads, 4)
pass2_push_kernel(const gs_segment* __restrict__ segs, const gs_chunk* __restrict__ chunks, int c0,
                  const int32_t* __restrict__ chunk_list, const gs_step_params* __restrict__ params, const float* __restrict__ seg_scale,
                  const uint32_t* __restrict__ flags, uint32_t flag_mask,
                  const uint64_t* __restrict__ peer_working, int p, int rank, uint8_t* mc) {
  gs::griddep_wait();  // the trust kernel's scales (PDL launch)
  if (*flags & flag_mask) return;  // lars.py:161-163
  const int c = chunk_list != nullptr ? chunk_list[c0 + blockIdx.x] : c0 + blockIdx.x;
  const gs_chunk ch = chunks[c];
  const gs_segment* sp = segs + ch.seg;
  const uint32_t sflags = sp->flags;
  Ctx cx;
  cx.u.load(params);
  cx.mul = params->mul;
  cx.wd = params->weight_decay;
  cx.m = params->momentum;
  const float s = seg_scale[ch.seg];
  uint16_t* w16 = sp->w16 + ch.start;
  const size_t woff = reinterpret_cast<const uint8_t*>(w16) -
                      reinterpret_cast<const uint8_t*>(peer_working[rank]);
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  const uint16_t* g = static_cast<const uint16_t*>(sp->g) + ch.start;
  if (decay)
    p2_push_chunk<POW2, true>(g, sp->w + ch.start, sp->v + ch.start, w16, ch.len, cx, s,
                              peer_working, p, rank, woff, mc);
  else
    p2_push_chunk<POW2, false>(g, sp->w + ch.start, sp->v + ch.start, w16, ch.len, cx, s,
                               peer_working, p, rank, woff, mc);
}

__global__ void peer_fence_kernel(const uint64_t* __restrict__ sig, int rank, int p, uint32_t epoch,
                                  const uint32_t* __restrict__ epoch_base) {
  epoch += *epoch_base;
  if (threadIdx.x < p) __threadfence_system();  // this GPU's earlier remote stores
  peer_barrier(sig, rank, p, 1, epoch);
}

}  // namespace

extern "C" {

int gs_rs_pass1(const uint64_t* wires, const void* own_wire, const uint64_t* sig, int rank, int p,
                const gs_segment* segs, const gs_chunk* chunks, int c0, int c1,
                const int32_t* chunk_list, const gs_step_params* params, uint32_t hint, const uint64_t* peer_partials,
                const uint64_t* peer_flags, uint32_t epoch, const uint32_t* epoch_base,
                int nblocks, void* stream) {
  GS_REQUIRE(p == 2 || p == 4 || p == 8, "gs_rs_pass1: p must be 2, 4 or 8 (got %d)", p);
  GS_REQUIRE(rank >= 0 && rank < p && c0 >= 0 && c1 >= c0 && nblocks >= 1,
             "gs_rs_pass1: bad arguments");
  GS_REQUIRE(wires && sig && segs && chunks && params && peer_partials && peer_flags && epoch_base,
             "gs_rs_pass1: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const uint8_t* ow = static_cast<const uint8_t*>(own_wire);
  const bool pow2 = hint & GS_HINT_POW2, raw = pow2 && (hint & GS_HINT_RAWFLAG),
             gnorm = hint & GS_HINT_GRADNORM, stage = (hint & GS_HINT_RS_STAGE) != 0;
  // every CTA waits for its peers at entry: the grid must be co-resident
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int nb = nblocks;
#define GS_RSP(P, PW, RW, GN)                                                                     \
  {                                                                                               \
    if (stage) {                                                                                  \
      auto k = rs_pass1_kernel<P, PW, RW, GN, true>;                                              \
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageBytes<P>);       \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, kStageBytes<P>);        \
      nb = min(nblocks, max(1, per_sm * sms));                                                    \
      k<<<nb, kThreads, kStageBytes<P>, s>>>(wires, ow, sig, rank, segs, chunks, c0, c1, chunk_list,  \
                                             params,                                              \
                                             peer_partials, peer_flags, epoch, epoch_base);       \
    } else {                                                                                      \
      auto k = rs_pass1_kernel<P, PW, RW, GN, false>;                                             \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);                     \
      nb = min(nblocks, max(1, per_sm * sms));                                                    \
      k<<<nb, kThreads, 0, s>>>(wires, ow, sig, rank, segs, chunks, c0, c1, chunk_list, params,       \
                                peer_partials,                                                    \
                                peer_flags, epoch, epoch_base);                                   \
    }                                                                                             \
  }
#define GS_RSP_P(P)                                      \
  if (raw) {                                             \
    if (gnorm) GS_RSP(P, true, true, true)               \
    else GS_RSP(P, true, true, false)                    \
  } else if (pow2) {                                     \
    if (gnorm) GS_RSP(P, true, false, true)              \
    else GS_RSP(P, true, false, false)                   \
  } else {                                               \
    if (gnorm) GS_RSP(P, false, false, true)             \
    else GS_RSP(P, false, false, false)                  \
  }
  if (p == 2) GS_RSP_P(2)
  else if (p == 4) GS_RSP_P(4)
  else GS_RSP_P(8)
#undef GS_RSP_P
#undef GS_RSP
  return gs_check_launch("gs_rs_pass1");
}

int gs_pass2_push(const gs_segment* segs, const gs_chunk* chunks, int c0, int c1,
                  const int32_t* chunk_list, const gs_step_params* params, uint32_t hint, const float* seg_scale,
                  const uint32_t* flags, uint32_t flag_mask, const uint64_t* peer_working, int p,
                  int rank, void* mc_working, void* stream) {
  GS_REQUIRE(c0 >= 0 && c1 >= c0 && p >= 1 && rank >= 0 && rank < p, "gs_pass2_push: bad arguments");
  if (c1 == c0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && seg_scale && flags && peer_working,
             "gs_pass2_push: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (hint & GS_HINT_POW2)
    e = gs_launch_pdl(pass2_push_kernel<true>, dim3(c1 - c0), dim3(kThreads), 0, s, segs, chunks, c0,
                      chunk_list, params, seg_scale, flags, flag_mask, peer_working, p, rank,
                      static_cast<uint8_t*>(mc_working));
  else
    e = gs_launch_pdl(pass2_push_kernel<false>, dim3(c1 - c0), dim3(kThreads), 0, s, segs, chunks,
                      c0, chunk_list, params, seg_scale, flags, flag_mask, peer_working, p, rank,
                      static_cast<uint8_t*>(mc_working));
  if (e != cudaSuccess) {
    gs_set_error("gs_pass2_push: %s", cudaGetErrorString(e));
    return GS_ECUDA;
  }
  return gs_check_launch("gs_pass2_push");
}

int gs_peer_fence(const uint64_t* sig, int rank, int p, uint32_t epoch, const uint32_t* epoch_base,
                  void* stream) {
  GS_REQUIRE(p >= 1 && p <= 32 && rank >= 0 && rank < p, "gs_peer_fence: bad arguments");
  if (p == 1) return GS_OK;
  GS_REQUIRE(sig && epoch_base, "gs_peer_fence: null pointer");
  peer_fence_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(sig, rank, p, epoch, epoch_base);
  return gs_check_launch("gs_peer_fence");
}

}  // extern "C"
