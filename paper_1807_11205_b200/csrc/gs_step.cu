// gs_step.cu — the native step executor: one C call launches a whole step.
//
// The pipeline's steps are short kernel sequences (p = 1: pass 1 -> trust
// -> pass 2; the sharded step: reduce-scatter + pass 1 -> fence -> trust ->
// pass 2 + push -> fence).  Issued from Python one ctypes call at a time the
// host needs longer than the device for the multi-GPU step (measured at
// p = 2: 0.30 ms per step against 0.15 ms of kernels), so the hot sequences
// are launched from here: one call, no per-kernel Python work, the same
// kernels in the same order as GradientPipeline's generator path (which
// stays for phase timing, NVTX ranges, the incremental API and the NCCL
// paths).  Under emulation (nranks = p ranks on one device) the rank-local
// kernels are launched per rank and every peer kernel once for all ranks.
#include "gs_common.cuh"

extern "C" {

int gs_batched_copy(const gs_copy* copies, int ncopies, void* stream);
int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, double* partials,
                  gs_ctl* ctl, uint32_t parity, const double* wsq, void* stream);
int gs_lars_trust(const gs_segment* segs, int nseg, int nchunk, const double* partials,
                  gs_step_params params, float* seg_scale, double* seg_out, gs_ctl* ctl,
                  uint32_t parity, const uint64_t* peer_ctl, int npeers, void* stream);
int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, const float* seg_scale,
                  const gs_ctl* ctl, uint32_t parity, uint32_t flag_mask, double* wsq,
                  void* stream);
int gs_rs_pass1(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* wires,
                const uint64_t* sig, const uint64_t* peer_partials, const uint64_t* peer_ctl,
                int b0, int b1, gs_step_params params, uint32_t hint, uint32_t parity,
                uint32_t epoch, int nblocks, void* stream);
int gs_pass2_push(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* peer_working,
                  int b0, int b1, int max_chunks, gs_step_params params, uint32_t hint,
                  uint32_t parity, uint32_t flag_mask, void* stream);
int gs_peer_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig, uint32_t epoch,
                  uint32_t epoch_inc, void* stream);
int gs_counter_add(uint32_t* counter, uint32_t inc, void* stream);
int gs_trust_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   uint32_t epoch, int nseg, int nchunk, gs_step_params params, uint32_t parity,
                   void* stream);
int gs_zero_update(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   const uint64_t* peer_working, uint32_t epoch, int nseg, int nchunk, int b0,
                   int b1, int max_chunks, gs_step_params params, uint32_t hint, uint32_t parity,
                   uint32_t flag_mask, void* stream);

#define GS_TRY(call)          \
  do {                        \
    const int rc_ = (call);   \
    if (rc_ != GS_OK) return rc_; \
  } while (0)

int gs_step_replicated(const gs_step_rank* r, int g_is_f16, gs_step_params params, uint32_t hint,
                       uint32_t parity, uint32_t flag_mask, void* stream) {
  GS_REQUIRE(r != nullptr, "gs_step_replicated: null rank");
  if (r->npack > 0) GS_TRY(gs_batched_copy(r->pack, r->npack, stream));
  GS_TRY(gs_lars_pass1(r->segs, r->chunks, 0, r->nchunk, g_is_f16, params, hint, r->partials,
                       r->ctl, parity, r->wsq_in, stream));
  GS_TRY(gs_lars_trust(r->segs, r->nseg, r->nchunk, r->partials, params, r->seg_scale,
                       r->seg_out, r->ctl, parity, nullptr, 0, stream));
  GS_TRY(gs_lars_pass2(r->segs, r->chunks, 0, r->nchunk, g_is_f16, params, hint, r->seg_scale,
                       r->ctl, parity, flag_mask, r->wsq_out, stream));
  return GS_OK;
}

int gs_step_zero(const gs_step_rank* ranks, int nranks, const gs_rank_ctx* ctx, int p,
                 const uint64_t* wires, const uint64_t* sig, const uint64_t* peer_partials,
                 const uint64_t* peer_ctl, const uint64_t* peer_working, int nbuckets,
                 int max_own, gs_step_params params, uint32_t hint, uint32_t parity,
                 uint32_t flag_mask, int nblocks, void* stream) {
  GS_REQUIRE(ranks != nullptr && ctx != nullptr && nranks >= 1 && nranks <= p && nbuckets >= 0,
             "gs_step_zero: bad arguments");
  for (int i = 0; i < nranks; ++i)
    if (ranks[i].npack > 0) GS_TRY(gs_batched_copy(ranks[i].pack, ranks[i].npack, stream));
  GS_TRY(gs_rs_pass1(ctx, nranks, p, wires, sig, peer_partials, peer_ctl, 0, nbuckets, params,
                     hint, parity, 1, nblocks, stream));
  // fence + trust + pass 2 with the working-weight push: one launch
  GS_TRY(gs_zero_update(ctx, nranks, p, sig, peer_working, 2, ranks[0].nseg, ranks[0].nchunk, 0,
                        nbuckets, max_own, params, hint, parity, flag_mask, stream));
  // the closing fence also advances every rank's epoch base by the step's 4
  GS_TRY(gs_peer_fence(ctx, nranks, p, sig, 3, 4, stream));
  return GS_OK;
}

}  // extern "C"
