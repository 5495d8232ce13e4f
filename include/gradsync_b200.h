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

#define GS_ABI_VERSION 3

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
  void* reserved2;
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

/* Per-step scalars, passed BY VALUE to every kernel of a step (kernel
 * parameter space): a step needs no host->device copy. */
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

/* Per-pipeline control block in device memory (zero-initialised).  The flag
 * words and the grad-norm arrival counter are double-buffered by step
 * parity: step k uses index k & 1, and its gs_lars_trust clears index
 * (k + 1) & 1 for the next step (the host read it after step k - 1). */
typedef struct gs_ctl {
  uint32_t flags[2];    /* GS_FLAG_* of the step with that parity */
  uint32_t counter[2];  /* gs_lars_trust's grad-norm arrival counter */
  uint32_t status;      /* peer-wait status, sticky: 0 = ok, else
                           0x80000000 | site << 20 | phase << 16 | peer << 8 | rank
                           of the first wait that timed out */
  uint32_t reserved[3];
  double grad_norm;     /* experiment.py:408-411 of the last step */
  double reserved2;
} gs_ctl; /* 48 bytes */

/* One rank of a peer-synchronised launch (the collectives and the fused
 * collective + LARS kernels).  A launch covers a device table of `nranks`
 * entries: 1 on a multi-GPU box (this GPU's rank), p when the p ranks of a
 * job are emulated on one device — CTA b then serves entry b / nb.  Built
 * and uploaded once per pipeline. */
typedef struct gs_rank_ctx {
  int32_t rank;                 /* 0 .. p-1 */
  int32_t reserved;
  uint64_t timeout_ns;          /* bound of every peer wait; 0 = 120 s */
  uint32_t* status;             /* where a timed-out wait is reported (usually
                                   &ctl->status); NULL = trap instead */
  const uint32_t* epoch_base;   /* device-resident epoch base added to every
                                   call's epoch (advanced by gs_counter_add), or NULL */
  const gs_segment* segs;       /* this rank's segment table (fused kernels) */
  const gs_chunk* chunks;       /* this rank's chunk table (fused kernels) */
  const int32_t* own_list;      /* chunk ids this rank folds / updates, bucket by bucket */
  const int32_t* own_off;       /* [nbuckets + 1]: bucket b owns own_list[own_off[b] .. own_off[b+1]) */
  gs_ctl* ctl;                  /* this rank's control block */
  const float* seg_scale;       /* trust scales (gs_pass2_push) */
  uint32_t* nonfinite;          /* ordered all-reduce / reduce-scatter: OR 1 here when a
                                   folded value is Inf/NaN (may be NULL) */
  void* red;                    /* gs_rs_pass1: base of this rank's reduced wire (the
                                   segments' g pointers lie in it; same layout as the
                                   raw wires the fold reads) */
  const double* partials;       /* gs_trust_fence: this rank's chunk partials */
  double* seg_out;              /* gs_trust_fence: per-segment norms / rates */
  uint32_t* seg_ready;          /* gs_zero_update: per-segment "scale published" epochs */
} gs_rank_ctx; /* 120 bytes */

/* One rank's buffers for the native step executor (gs_step_*): a HOST
 * struct (the executor reads it on the host and launches from it). */
typedef struct gs_step_rank {
  const gs_copy* pack;          /* optional pack table run before the step (device), or NULL */
  int32_t npack;
  int32_t nseg;
  const gs_segment* segs;       /* device segment / chunk tables */
  const gs_chunk* chunks;
  int32_t nchunk;
  int32_t reserved;
  double* partials;             /* device scratch of the LARS passes */
  float* seg_scale;
  double* seg_out;
  gs_ctl* ctl;
  const double* wsq_in;         /* replicated step: w^2 carried into pass 1 (or NULL) */
  double* wsq_out;              /* replicated step: pass 2's w^2 for the next step (or NULL) */
  uint32_t* epoch_base;         /* sharded step: the rank's device epoch base */
} gs_step_rank; /* 96 bytes */

/* Host-side launch hints: which specialised pass-1/pass-2 kernel may be used.
 * A hint is a promise about the params of the launch; 0 is always correct
 * (generic kernel, per-element IEEE division). */
#define GS_HINT_POW2 1u       /* g/div1/div2 == g*mul exactly: every active
                                 divisor is a power of two and (fp32 input) no
                                 divisor is active, or (fp16 input) div1 <= 2^100 */
#define GS_HINT_RAWFLAG 2u    /* fp16 input, GS_HINT_POW2 and mul <= 1: a value is
                                 non-finite iff its binary16 exponent is all ones */
#define GS_HINT_GRADNORM 4u   /* must equal (params.mode & GS_MODE_GRADNORM) != 0 */

int gs_abi_version(void);
const char* gs_last_error(void);
int gs_device_sm_count(int device);
/* Number of kernels this library has launched so far in the process (every
 * launch site counts once per kernel; bench.py's gpu_launches evidence). */
int64_t gs_kernel_launches(void);

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

/* ---- peer collectives (gs_collective.cu) -------------------------------
 * Every entry point below takes `ranks` / `nranks` (gs_rank_ctx) and is
 * called on every rank with otherwise identical arguments:
 *   bufs / sig / peer_*  device arrays of p peer-mapped base pointers (NVLink
 *          on a box; plain local pointers when ranks are emulated), entry
 *          [rank] = that rank's own; sig areas are zero-initialised uint32 of
 *          >= 2 * nblocks * p words;
 *   epoch  nonzero, strictly increasing per call on a given sig area (plus
 *          *ranks[i].epoch_base, so a step's calls can be replayed after the
 *          caller advances the base with gs_counter_add);
 *   nblocks  CTAs per rank; clamped so every rank's CTAs are co-resident.
 * A wait that exceeds ranks[i].timeout_ns reports through ranks[i].status
 * and drains instead of hanging the GPU. */

/* Bit-exact all-reduce of one binary16 bucket [offset, offset + n) of every
 * rank's (double-buffered) wire: the reference's pairwise tree
 * (fold_f16_tree, collectives.py:273-283) with the bytes of a ring (each rank
 * folds its slice from every peer's raw values; tcp.py:122-130 is the same
 * design over TCP).  push = 0: the slices are then gathered by peer loads
 * after a barrier; push = 1: the owner stores its folded slice into every
 * peer as it folds, one exit barrier.  Same result bit for bit.  p <= 8. */
int gs_ordered_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* sig, int64_t offset, int64_t n, uint32_t epoch,
                             int nblocks, int push, void* stream);

/* fp32 form for the reference's own fp32 wire (run_experiment fuses fp32
 * gradients, experiment.py:282-301, 368-399): every element is the ascending
 * left fold b0 + b1 + ... + b(p-1) in fp32 (fold_ascending,
 * collectives.py:261-270; ring and hierarchical give this same fold, the
 * mean's division by float32(p) is the consumer's: LARS pass 1).  n and
 * offset in fp32 elements; otherwise the contract of the binary16 kernel. */
int gs_ordered_allreduce_f32(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* sig, int64_t offset, int64_t n, uint32_t epoch,
                             int nblocks, int push, void* stream);

/* The same all-reduce over Topology(p, k)'s two levels (
 * hierarchical_schedule, collectives.py:183-235): an intra-group
 * reduce-scatter (each member folds its slice over the group's k raw
 * copies), an inter-group fold of each sub-slice over the p/k same-offset
 * group partials, then the all-gather.  For power-of-two k the reference's
 * rank tree factors exactly this way, so the result equals
 * gs_ordered_allreduce_f16's bit for bit.  push != 0: the rank that folds a
 * final sub-slice stores it into every rank and one exit barrier replaces
 * the gather (same bits).  Signal areas need >= 3 * nblocks * p words.
 * k in {2, 4, 8}, p <= 8. */
/* One-shot form of gs_ordered_allreduce_f16 for small buckets (same bits):
 * every rank stores its raw bucket into slot [parity][rank] (cap elements
 * each) of every rank's `inbox` (device table of p inbox base addresses),
 * one barrier, then folds its own p slots in the reference's tree order into
 * its buffer.  One barrier instead of two; (p-1) x S bytes out per rank.
 * Consecutive one-shot calls on the same inboxes must alternate parity.
 * n <= cap. */
int gs_oneshot_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* inbox, const uint64_t* sig, int64_t offset, int64_t n,
                             int64_t cap, uint32_t epoch, int nblocks, uint32_t parity,
                             void* stream);

/* LL form of the same all-reduce (no fence, no barrier): every 4 bytes of
 * payload travel as one 8-byte word {payload, epoch} into slot [parity][rank]
 * (cap / 2 words) of every rank's inbox; each rank polls its own slots until
 * every word carries this call's epoch, folds in the reference's tree order
 * and writes its buffer.  Same bits; 2 x (p-1) x S bytes out per rank.
 * Whole 8-element vectors only (n % 8 == 0, offset % 8 == 0, n <= cap);
 * consecutive LL / one-shot calls on the same inboxes alternate parity. */
int gs_ll_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                        const uint64_t* inbox, int64_t offset, int64_t n, int64_t cap,
                        uint32_t epoch, int nblocks, uint32_t parity, void* stream);

int gs_hier_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, int k,
                          const uint64_t* bufs, const uint64_t* sig, int64_t offset, int64_t n,
                          uint32_t epoch, int nblocks, int push, void* stream);

/* Reduce-scatter half of the above with explicit slices: rank r folds
 * elements [bounds[r], bounds[r+1]) (device int64 array of p + 1 offsets)
 * of every peer's buffer into its own, in the reference's tree order.  Used
 * by the sharded (ZeRO-1) update with separate collectives. */
int gs_ordered_reduce_scatter_f16(const gs_rank_ctx* ranks, int nranks, int p,
                                  const uint64_t* bufs, const uint64_t* sig, const int64_t* bounds,
                                  uint32_t epoch, int nblocks, void* stream);

/* All-gather of byte ranges over peer memory: rank r owns bytes
 * [bounds[r], bounds[r+1]) of its buffer; every rank copies the other ranks'
 * ranges from their buffers (entry and exit barriers).  Gathers the LARS
 * chunk partials, the binary16 working weights and (gather_state) the
 * sharded masters / velocities. */
int gs_ordered_allgather(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                         const uint64_t* sig, const int64_t* bounds, uint32_t epoch, int nblocks,
                         void* stream);

/* *counter += inc on the device (stream-ordered). */
int gs_counter_add(uint32_t* counter, uint32_t inc, void* stream);

/* ---- collective + LARS fused (sharded update, gs_fused.cu) ------------- */

/* Reduce-scatter fused with LARS pass 1 (replaces the reduce-scatter +
 * gs_lars_pass1 + the all-gather of the chunk partials; reference:
 * collectives.py:273-283 fold_f16_tree, then lars.py:142-177 norms).  After an
 * entry barrier, each rank takes its owned chunks of buckets [b0, b1)
 * (ranks[i].own_list / own_off; the segments' g pointers lie in
 * ranks[i].red), folds every peer's raw binary16 values of the chunk
 * (wires[q], never written) in the reference's tree order, stores the folded
 * chunk in its reduced wire, reduces
 * it to fp64 partials and STORES them into every peer's partials
 * (peer_partials[q], 3 doubles at the chunk's index); the step flags are
 * OR-ed into every peer's gs_ctl.flags[parity] (peer_ctl[q]).  p in {2,4,8}. */
int gs_rs_pass1(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* wires,
                const uint64_t* sig, const uint64_t* peer_partials, const uint64_t* peer_ctl,
                int b0, int b1, gs_step_params params, uint32_t hint, uint32_t parity,
                uint32_t epoch, int nblocks, void* stream);

/* LARS pass 2 over each rank's owned chunks of buckets [b0, b1) (one CTA
 * per chunk, grid = nranks * max_chunks where max_chunks >= every rank's
 * owned count) that also stores each updated binary16 working weight into
 * every peer's working arena (peer_working[q] = peer q's base; the
 * segments' w16 lie in peer_working[rank]).  Replaces gs_lars_pass2 + the
 * all-gather of the working weights (lars.py:178-181).  Launched as a
 * programmatic dependent of gs_lars_trust. */
int gs_pass2_push(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* peer_working,
                  int b0, int b1, int max_chunks, gs_step_params params, uint32_t hint,
                  uint32_t parity, uint32_t flag_mask, void* stream);

/* One CTA per rank: this rank's remote stores from earlier kernels on the
 * stream are visible to every peer, and every peer's to this rank.
 * epoch_inc != 0: afterwards add it to the rank's device epoch base (the
 * step's last kernel advances the base for the next step). */
int gs_peer_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig, uint32_t epoch,
                  uint32_t epoch_inc, void* stream);

/* gs_peer_fence(epoch) followed by gs_lars_trust in ONE launch (the
 * sharded step's middle): the first nranks CTAs fence and run the peer
 * barrier (one per rank, as gs_peer_fence), then publish `epoch` in
 * ctl->counter[0]; the other nranks x (nseg + 1) CTAs wait for their rank's
 * word and run the trust kernel's CTAs over the rank's segs / partials /
 * seg_scale / seg_out / ctl from the gs_rank_ctx table (same order, same
 * bits).  pass 2 may be PDL-launched behind it. */
int gs_trust_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   uint32_t epoch, int nseg, int nchunk, gs_step_params params, uint32_t parity,
                   void* stream);

/* gs_trust_fence and gs_pass2_push in ONE launch (the whole second half of
 * the sharded step): fence CTAs, then trust CTAs (each publishes its
 * segment's epoch in ctx.seg_ready[s] after the scale), then pass-2 CTAs
 * (max_chunks per rank) that wait for their chunk's segment.  Every wait is
 * on CTAs earlier in the grid, so it cannot deadlock.  Same bits. */
int gs_zero_update(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   const uint64_t* peer_working, uint32_t epoch, int nseg, int nchunk, int b0,
                   int b1, int max_chunks, gs_step_params params, uint32_t hint, uint32_t parity,
                   uint32_t flag_mask, void* stream);

/* ---- native step executor (gs_step.cu) ---------------------------------
 * One call launches a whole step — the same kernels, in the same order, as
 * the pipeline's per-kernel path, without per-kernel host work. */

/* p = 1 / replicated update: [pack] -> gs_lars_pass1 -> gs_lars_trust ->
 * gs_lars_pass2 (experiment.py:403-412 after the all-reduce). */
int gs_step_replicated(const gs_step_rank* rank, int g_is_f16, gs_step_params params,
                       uint32_t hint, uint32_t parity, uint32_t flag_mask, void* stream);

/* The sharded (ZeRO-1) step in fused kernels for `nranks` ranks (1 on a box,
 * p when emulated; ranks = host array, ctx = device gs_rank_ctx table):
 * [pack per rank] -> gs_rs_pass1 -> gs_zero_update (fence + trust +
 * pass 2 with the working-weight push) -> gs_peer_fence (which adds 4 to
 * every rank's epoch base).  Epochs
 * 1, 2, 3 of the step; max_own >= every rank's owned chunk count. */
int gs_step_zero(const gs_step_rank* ranks, int nranks, const gs_rank_ctx* ctx, int p,
                 const uint64_t* wires, const uint64_t* sig, const uint64_t* peer_partials,
                 const uint64_t* peer_ctl, const uint64_t* peer_working, int nbuckets,
                 int max_own, gs_step_params params, uint32_t hint, uint32_t parity,
                 uint32_t flag_mask, int nblocks, void* stream);

/* ---- LARS (lars.py:142-181) fused over a segment table ---------------- */

/* Pass 1 over `nchunk` chunks starting at chunk index `chunk0`: widen (fp16
 * grads) / mean / unscale per params.mode, OR the non-finite flags into
 * ctl->flags[parity], and write per-chunk fp64 partials {sum w^2, sum eff^2,
 * sum g^2} (lars.py:145-146, 169-172; experiment.py:408-411) to
 * partials[3*chunk + k].  g_is_f16 selects the gradient element type.
 * wsq (optional, nchunk doubles): per-chunk sum w^2 left by gs_lars_pass2 of
 * the previous step over the same masters; a non-NaN entry replaces the
 * chunk's w^2 accumulation (same order, same bits).  Pass NULL whenever the
 * masters may have changed since (a load, a checkpoint restore). */
int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, double* partials,
                  gs_ctl* ctl, uint32_t parity, const double* wsq, void* stream);

/* One CTA per segment: fold the chunk partials in a fixed order, take the
 * fp64 norms, local = eta*||w|| / (||eff|| + eps) or 1.0 (lars.py:142-150,
 * 173-176) and seg_scale[s] = float32(local * gamma) (lars.py:177).  seg_out
 * (nseg x 4 doubles) receives {||w||, ||eff||, local, sum g^2}; with
 * GS_MODE_GRADNORM one more CTA writes ctl->grad_norm = sqrt of the sum of
 * all nchunk chunks' g^2 (experiment.py:408-411).  Clears
 * ctl->flags/counter[parity ^ 1] for the next step.  peer_ctl (npeers device
 * pointers, sharded update with separate collectives): OR every rank's
 * flags[parity] into this rank's, so a non-finite value anywhere rejects the
 * step everywhere.  Launched as a programmatic dependent of pass 1. */
int gs_lars_trust(const gs_segment* segs, int nseg, int nchunk, const double* partials,
                  gs_step_params params, float* seg_scale, double* seg_out, gs_ctl* ctl,
                  uint32_t parity, const uint64_t* peer_ctl, int npeers, void* stream);

/* Pass 2: if (ctl->flags[parity] & flag_mask) do nothing (lars.py:161-163 —
 * the step is rejected with no mutation).  Otherwise per element
 *   eff = g  or  g + wd*w                 (lars.py:169-172)
 *   v   = momentum*v + seg_scale[s]*eff   (lars.py:178)
 *   w   = w - v                           (lars.py:179)
 *   w16 = f32_to_f16(w)                   (lars.py:180)
 * Chunks are visited in reverse order (L2 reuse after pass 1).  wsq
 * (optional): receives, per LARS chunk, the sum of the updated w^2 in pass
 * 1's order (NaN where pass 1's vector order cannot be reproduced) for the
 * next step's gs_lars_pass1. */
int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, const float* seg_scale,
                  const gs_ctl* ctl, uint32_t parity, uint32_t flag_mask, double* wsq,
                  void* stream);

/* Write `nbytes` of 0 to dst with a kernel (L2 flush helper). */
int gs_fill_zero(void* dst, int64_t nbytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GRADSYNC_B200_H */
