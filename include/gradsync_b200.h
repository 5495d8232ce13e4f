/*
 * gradsync_b200.h — C ABI of the B200 gradient-pipeline library
 * (libgradsync_b200.so, built from paper_1807_11205_b200/csrc/).
 *
 * The reference (gradsync, pkg/src/gradsync) is pure Python + numpy and has no
 * FFI layer; its drop-in boundary is the Python API re-exported by
 * pkg/src/gradsync/__init__.py:3-70.  Every entry point below replaces the
 * numpy arithmetic behind one of those Python functions; the Python shims in
 * paper_1807_11205_b200/*.py keep the reference signatures, validation and
 * error messages and call these through ctypes.
 *
 * Conventions
 *   - All data pointers are CUDA device pointers (or peer-mapped device
 *     pointers for the *_slots entry points).  Tables (gs_segment, gs_chunk,
 *     gs_copy, slot pointer arrays, gs_step_params) also live in device memory;
 *     the caller builds and uploads them once and reuses them.
 *   - `stream` is a cudaStream_t passed as void*.  Every call is asynchronous
 *     on that stream, allocates nothing and never synchronises.
 *   - Return value: 0 on success, negative on a bad argument (GS_EINVAL) or a
 *     launch error (GS_ECUDA); gs_last_error() then holds a message.
 *   - fp16 data is carried as uint16_t binary16 bit patterns, exactly like the
 *     reference (halfprec.py:3-7).  Every narrowing is IEEE round-to-nearest-
 *     even with overflow to +-Inf and every NaN canonicalised to 0x7E00
 *     (halfprec.py:40-85).
 *   - No FMA contraction anywhere an fp32 result is observable: products and
 *     sums are rounded separately, matching numpy's separate ufunc calls.
 */
#ifndef GRADSYNC_B200_H
#define GRADSYNC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 1

#define GS_OK 0
#define GS_EINVAL (-1)
#define GS_ECUDA (-2)

/* gs_segment.flags — same bit meaning as the LARS v1 checkpoint flag byte
 * (lars.py:186-188 / pkg/README.md:167-173). */
#define GS_SEG_DECAY_EXEMPT 1u
#define GS_SEG_LARS_ENABLED 2u

/* gs_step_params.mode bits */
#define GS_MODE_DIV1 1u        /* divide widened gradient by div1 (mean over p) */
#define GS_MODE_DIV1_POW2 2u   /* div1 is a power of two: multiply by rcp1 (bit-identical) */
#define GS_MODE_DIV2 4u        /* divide by div2 (loss-scale unscale) */
#define GS_MODE_DIV2_POW2 8u   /* div2 is a power of two: multiply by rcp2 */
#define GS_MODE_DECAY 16u      /* cfg.weight_decay != 0.0 (lars.py:169) */
#define GS_MODE_GRADNORM 32u   /* also accumulate sum(g^2) for the grad-norm metric */

/* device flag word bits written by gs_lars_pass1 / gs_nonfinite_* */
#define GS_FLAG_SCALED_NONFINITE 1u   /* LossScale.update finite test (halfprec.py:210) */
#define GS_FLAG_GRAD_NONFINITE 2u     /* lars_step finite gate (lars.py:161-163) */

/* One parameter group (lars.py:92-125) as seen by the fused kernels. */
typedef struct gs_segment {
  const void* g;        /* gradient: fp16 bits (uint16) or fp32, per call flag */
  float* w;             /* fp32 master weights */
  float* v;             /* fp32 velocity */
  uint16_t* w16;        /* binary16 working copy */
  int64_t n;            /* element count */
  int32_t chunk_begin;  /* first chunk of this segment in the chunk table */
  int32_t chunk_count;  /* number of chunks of this segment */
  uint32_t flags;       /* GS_SEG_* */
  uint32_t reserved;
  void* gcopy;          /* optional: pass 1 also copies the raw fp16 gradient
                           chunk here (the fused packer), or NULL */
} gs_segment; /* 64 bytes */

/* A contiguous piece [start, start+len) of segment `seg`; len <= 65536. */
typedef struct gs_chunk {
  int64_t start;
  int32_t seg;
  int32_t len;
} gs_chunk; /* 16 bytes */

/* One byte range copy for the fusion packer (fusion.py:83-94). */
typedef struct gs_copy {
  const void* src;
  void* dst;
  int64_t nbytes;
} gs_copy; /* 24 bytes */

/* Per-step scalars, in device memory so a captured CUDA graph can be replayed
 * with a new loss scale / learning rate by rewriting this struct. */
typedef struct gs_step_params {
  double eta;           /* LarsConfig.eta (lars.py:76) */
  double epsilon;       /* LarsConfig.epsilon */
  double gamma;         /* Schedule.lr(step) (lars.py:165), fp64 */
  float weight_decay;   /* float32(cfg.weight_decay) (lars.py:166) */
  float momentum;       /* float32(cfg.momentum) (lars.py:167) */
  float div1, rcp1;     /* mean divisor float32(p) (collectives.py:268-269) */
  float div2, rcp2;     /* unscale divisor float32(scale) (halfprec.py:234) */
  uint32_t mode;        /* GS_MODE_* */
  float mul;            /* rcp1*rcp2 when both divisions are exact power-of-two
                           scalings (see GS_HINT_POW2), else unused */
} gs_step_params; /* 56 bytes */

/* Host-side launch hints: which specialised pass-1/pass-2 kernel may be used.
 * A hint is a promise about the contents of *params at execution time; 0 is
 * always correct (generic kernel, per-element IEEE division). */
#define GS_HINT_POW2 1u       /* g/div1/div2 == g*mul exactly: every active
                                 divisor is a power of two and (fp32 input) no
                                 divisor is active, or (fp16 input) div1 <= 2^100 */
#define GS_HINT_RAWFLAG 2u    /* fp16 input, GS_HINT_POW2 and mul <= 1: a value is
                                 non-finite iff its binary16 exponent is all ones */
#define GS_HINT_GRADNORM 4u   /* must equal (params->mode & GS_MODE_GRADNORM) != 0 */
#define GS_HINT_RS_STAGE 16u  /* gs_rs_pass1: stage a chunk's peer vectors in shared
                                 memory with cp.async (all in flight at once) instead
                                 of register loads per vector (measured slower) */
#define GS_HINT_NO_BULK 8u    /* fp16 pass 1: use the register-staged kernel instead of
                                 the TMA (cp.async.bulk) pipelined persistent kernel */

int gs_abi_version(void);
const char* gs_last_error(void);
int gs_device_sm_count(int device);

/* ---- halfprec (halfprec.py) -------------------------------------------- */

/* h[i] = f32_to_f16(x[i] * scale)  (halfprec.py:108-121; with scale == 1 the
 * multiply is the identity).  If nonfinite != NULL, OR 1 into *nonfinite when
 * any h[i] is Inf/NaN. */
int gs_f32_to_f16(const float* x, uint16_t* h, int64_t n, float scale,
                  uint32_t* nonfinite, void* stream);

/* x[i] = f16_to_f32(h[i]), exact (halfprec.py:88-105, 124-132). */
int gs_f16_to_f32(const uint16_t* h, float* x, int64_t n, void* stream);

/* y[i] = f16_to_f32(f32_to_f16(x[i])) (halfprec.py:135-137). */
int gs_quantize_f32(const float* x, float* y, int64_t n, void* stream);

/* out[i] = float32(g[i]) / float32(scale), IEEE division (halfprec.py:230-234). */
int gs_unscale_f32(const float* g, float* out, int64_t n, float scale, void* stream);

/* OR `bit` into *flag if any element of any tensor is non-finite
 * (LossScale.update, halfprec.py:209-210; lars_step gate, lars.py:161-163).
 * ptrs/lens are device arrays of ntensors entries; max_len (host value) is the
 * longest length and sizes the grid; is_f16 selects uint16 binary16 vs fp32. */
int gs_nonfinite(const uint64_t* ptrs, const int64_t* lens, int ntensors, int64_t max_len,
                 int is_f16, uint32_t* flag, uint32_t bit, void* stream);

/* ---- fusion (fusion.py) ------------------------------------------------ */

/* Batched byte copy: copies[i].src -> copies[i].dst for ncopies entries
 * (device table).  Used for FusionBuffer._emit (fusion.py:83-94) and for the
 * fused pipeline's bucket packer.  Entries may have any alignment. */
int gs_batched_copy(const gs_copy* copies, int ncopies, void* stream);

/* ---- in-order folds (collectives.py:261-283) -------------------------- */

/* out = slots[0] + slots[1] + ... + slots[p-1] as an ascending fp32 left fold;
 * if mean, out /= float32(p) (fold_ascending, collectives.py:261-270).
 * slots: device array of p device (or peer) pointers; each slot is offset by
 * `offset` elements.  out may alias slots[0]. */
int gs_fold_f32(const uint64_t* slots, int p, int64_t offset, float* out, int64_t n,
                int mean, void* stream);

/* Pairwise-tree fold of binary16 patterns with widen-add-narrow combines:
 * level pairs (i, i+1), odd tail carried (fold_f16_tree, collectives.py:273-283).
 * out may alias slots[0].  If nonfinite != NULL, OR 1 into *nonfinite when any
 * output element is Inf/NaN. */
int gs_fold_f16_tree(const uint64_t* slots, int p, int64_t offset, uint16_t* out,
                     int64_t n, uint32_t* nonfinite, void* stream);

/* Bit-exact all-reduce of one binary16 bucket over NVLink peer memory: the
 * reference's pairwise tree (fold_f16_tree, collectives.py:273-283) with the
 * bytes of a ring (reduce-scatter by peer loads, then all-gather by peer
 * loads; tcp.py:122-130 is the same design over TCP).  Call on every rank
 * with the same arguments except `rank`:
 *   bufs   device array of p peer-mapped base pointers of the (symmetric)
 *          wire buffers, bufs[rank] = this rank's own;
 *   sig    device array of p peer-mapped pointers to zero-initialised uint32
 *          signal areas of >= 2 * nblocks * p words each;
 *   offset, n  the bucket (elements) inside every wire;
 *   epoch  nonzero, strictly increasing per call on a given sig area; with
 *          epoch_base != NULL the kernel uses epoch + *epoch_base instead, so
 *          a captured CUDA graph stays valid when the caller advances the
 *          device-resident base between replays (gs_counter_add);
 *   nblocks  grid size; all CTAs must be co-resident (<= SMs).
 * The wire must be double-buffered across consecutive calls on the same
 * range (the kernel has no exit barrier).  p <= 8. */
int gs_ordered_allreduce_f16(const uint64_t* bufs, const uint64_t* sig, int rank, int p,
                             int64_t offset, int64_t n, uint32_t epoch,
                             const uint32_t* epoch_base, int nblocks, uint32_t* nonfinite,
                             void* stream);

/* Same contract and result as gs_ordered_allreduce_f16, push form: the
 * owner of a slice stores the folded slice into every peer's buffer as it
 * folds (remote stores), then one exit barrier; no gather phase.  The wire
 * must still be double-buffered across calls. */
int gs_ordered_allreduce_push_f16(const uint64_t* bufs, const uint64_t* sig, int rank, int p,
                                  int64_t offset, int64_t n, uint32_t epoch,
                                  const uint32_t* epoch_base, int nblocks, uint32_t* nonfinite,
                                  void* stream);

/* Reduce-scatter half of the above with explicit slices: rank r folds
 * elements [bounds[r], bounds[r+1]) (device int64 array of p + 1 offsets)
 * of every peer's buffer into its own, in the reference's tree order.  Used
 * by the sharded (ZeRO-1) update, whose slices follow chunk boundaries. */
int gs_ordered_reduce_scatter_f16(const uint64_t* bufs, const uint64_t* sig, int rank, int p,
                                  const int64_t* bounds, uint32_t epoch, const uint32_t* epoch_base,
                                  int nblocks, uint32_t* nonfinite, void* stream);

/* All-gather of byte ranges over peer memory: rank r owns bytes
 * [bounds[r], bounds[r+1]) of its buffer; every rank copies the other ranks'
 * ranges from their buffers (entry and exit barriers).  Used to gather the
 * LARS chunk partials and the binary16 working weights of the sharded
 * update. */
int gs_ordered_allgather(const uint64_t* bufs, const uint64_t* sig, int rank, int p,
                         const int64_t* bounds, uint32_t epoch, const uint32_t* epoch_base,
                         int nblocks, void* stream);

/* *counter += inc on the device (stream-ordered; graph-capturable). */
int gs_counter_add(uint32_t* counter, uint32_t inc, void* stream);

/* ---- collective + LARS fused (sharded update, gs_fused.cu) ------------- */

/* Reduce-scatter fused with LARS pass 1 (replaces gs_ordered_reduce_scatter_f16
 * + gs_lars_pass1 + the all-gather of the chunk partials; reference:
 * collectives.py:273-283 fold_f16_tree then lars.py:142-177 norms).  After an
 * entry barrier, chunks [c0, c1) of the local chunk table — this rank's
 * chunks of one bucket — are folded from every peer's wire (wires[q] = peer
 * q's base, the segment's g pointers lie in wires[rank]) in the reference's
 * tree order, stored into the local wire, and reduced to fp64 partials that
 * are STORED into every peer's partials array (peer_partials[q], 3 doubles
 * per chunk at the chunk's global index); the step flags are OR-ed into every
 * peer's flag word (peer_flags[q]).  Every rank must call it (also with
 * c0 == c1) with the same epoch; p in {2, 4, 8}.  A non-null chunk_list
 * (device int32) makes the chunks chunk_list[c0 .. c1-1] (the rank's owned
 * chunks of several buckets: one launch, one entry barrier).
 * own_wire == NULL: pull form, as above.  own_wire != NULL: inbox form —
 * every rank's packer already STORED its raw values of this rank's slices
 * into this rank's inboxes (wires[q] = this rank's inbox holding rank q's
 * values, wire-shaped); the fold then reads local memory only, own_wire is
 * this rank's wire base (the segments' g pointers lie in it). */
int gs_rs_pass1(const uint64_t* wires, const void* own_wire, const uint64_t* sig, int rank, int p,
                const gs_segment* segs, const gs_chunk* chunks, int c0, int c1,
                const int32_t* chunk_list, const gs_step_params* params, uint32_t hint, const uint64_t* peer_partials,
                const uint64_t* peer_flags, uint32_t epoch, const uint32_t* epoch_base,
                int nblocks, void* stream);

/* LARS pass 2 over chunks [c0, c1) (binary16 gradients; with a non-null
 * chunk_list, over chunks chunk_list[c0 .. c1-1]) that also stores each
 * updated binary16 working weight into every peer's working arena
 * (peer_working[q] = peer q's base; the segments' w16 lie in
 * peer_working[rank]).  mc_working != NULL: the NVLS multicast address of
 * peer_working[rank]'s window (same offsets) — one multimem store per vector
 * reaches every rank.  Replaces gs_lars_pass2 + the all-gather of the
 * working weights (lars.py:178-181).  Launched as a programmatic dependent of
 * gs_lars_trust. */
int gs_pass2_push(const gs_segment* segs, const gs_chunk* chunks, int c0, int c1,
                  const int32_t* chunk_list, const gs_step_params* params, uint32_t hint, const float* seg_scale,
                  const uint32_t* flags, uint32_t flag_mask, const uint64_t* peer_working, int p,
                  int rank, void* mc_working, void* stream);

/* One-CTA barrier: this GPU's remote stores from earlier kernels on the
 * stream are visible to every peer, and every peer's to this GPU. */
int gs_peer_fence(const uint64_t* sig, int rank, int p, uint32_t epoch, const uint32_t* epoch_base,
                  void* stream);

/* ---- LARS (lars.py:142-181) fused over a segment table ---------------- */

/* Pass 1 over `nchunk` chunks starting at chunk index `chunk0`: widen (fp16
 * grads) / mean / unscale per params->mode, OR the non-finite flags, and write
 * per-chunk fp64 partials {sum w^2, sum eff^2, sum g^2} (lars.py:145-146,
 * 169-172; experiment.py:408-411) to partials[3*chunk + k].  g_is_f16 selects
 * the gradient element type for every segment. */
int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, uint32_t hint, double* partials,
                  uint32_t* flags, void* stream);

/* gs_lars_pass1 fused with gs_lars_trust.  counters: device uint32[nseg + 1],
 * zero before the first chunk of a step is launched (reset together with
 * the flags).  The last CTA to finish a segment folds that segment's
 * partials (same fixed order as gs_lars_trust) and writes seg_scale /
 * seg_out; the last segment to finish (of nseg_active segments that own at
 * least one chunk) fills the empty segments and writes *grad_norm_out.  May
 * be called over several disjoint chunk ranges per step (e.g. one per
 * bucket as its all-reduce lands). */
int gs_lars_pass1_trust(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                        int chunk0, int nchunk, int g_is_f16, const gs_step_params* params,
                        uint32_t hint, double* partials, uint32_t* flags, uint32_t* counters,
                        float* seg_scale, double* seg_out, double* grad_norm_out, void* stream);

/* Per segment (one CTA each): fold the chunk partials in a fixed order (the
 * same order as gs_lars_pass1_trust), take the fp64 norms,
 * local = eta*||w|| / (||eff|| + eps) or 1.0 (lars.py:142-150, 173-176) and
 * seg_scale[s] = float32(local * gamma) (lars.py:177).  seg_out (nseg x 4
 * doubles) receives {||w||, ||eff||, local, sum g^2}; grad_norm_out (optional)
 * receives sqrt of the sum of per-segment g^2 in segment order
 * (experiment.py:408-411) and then needs `counter`, one zeroed uint32.
 * peer_flags (npeers device pointers, sharded update): OR every rank's step
 * flags into *flags so a non-finite value anywhere rejects the step
 * everywhere; npeers = 0 otherwise. */
int gs_lars_trust(const gs_segment* segs, int nseg, const double* partials,
                  const gs_step_params* params, float* seg_scale, double* seg_out,
                  double* grad_norm_out, uint32_t* counter, const uint64_t* peer_flags,
                  int npeers, uint32_t* flags, void* stream);

/* Pass 2: if (*flags & flag_mask) do nothing (lars.py:161-163 — the step is
 * rejected with no mutation).  Otherwise per element
 *   eff = g  or  g + wd*w                 (lars.py:169-172)
 *   v   = momentum*v + seg_scale[s]*eff   (lars.py:178)
 *   w   = w - v                           (lars.py:179)
 *   w16 = f32_to_f16(w)                   (lars.py:180)
 */
int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, uint32_t hint,
                  const float* seg_scale, const uint32_t* flags, uint32_t flag_mask,
                  void* stream);

/* Write `nbytes` of 0 to dst with a kernel (L2 flush helper / flag reset). */
int gs_fill_zero(void* dst, int64_t nbytes, void* stream);

/* gs_lars_trust fused into gs_lars_pass2 (one launch over the whole chunk
 * table): every CTA folds its own segment's chunk partials (same order as
 * gs_lars_trust, so every CTA of a segment derives the same fp32 scale)
 * while its chunk is prefetched into L2; the segment's first CTA writes
 * seg_scale/seg_out, and the last of those (of nseg_active segments owning a
 * chunk; arrival counter, one zeroed uint32) writes the empty segments and
 * *grad_norm_out.  Nothing is written
 * when (*flags & flag_mask) (lars.py:161-163). */
int gs_lars_pass2_trust(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                        int chunk0, int nchunk, int g_is_f16, const gs_step_params* params, uint32_t hint,
                        const double* partials, float* seg_scale, double* seg_out,
                        double* grad_norm_out, uint32_t* counter, const uint32_t* flags,
                        uint32_t flag_mask, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GRADSYNC_B200_H */
