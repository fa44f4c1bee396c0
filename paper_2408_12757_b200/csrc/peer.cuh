// Fused row-parallel GEMM + AllReduce over peer memory (
// the paper's collectives were MSCCL++ SM-constrained kernels,
// PAPER.md:612-614 gives the network operation its own SM budget).
//
// Every rank holds one symmetric buffer (same layout on all ranks; mapped into the
// other ranks' address spaces through CUDA IPC, or plain pointers in an emulated
// group).  A row-parallel GEMM whose output must be summed over the TP group (the
// O2 row-parallel projection, the Down projection) runs the
// EPI_PEER epilogue: each 128x256 output block has an owner rank (block % N) and
// the epilogue stores its bf16 partial block straight into the owner's staging
// slot [src rank][owned block] and bumps the owner's arrival flag (reduce-scatter
// fused into the GEMM: the transfer of block b overlaps the math of the following
// tiles).  The owner's peer_reduce kernel (network stream / partition) waits on each
// owned block's flag, sums the N partials in rank order in fp32 with one bf16
// rounding (the same arithmetic as the emulated NF_AR_F32 AllReduce), and pushes
// the block to every rank's result region (all-gather), bumping their `done`
// counters; it ends when its own `done` counter has seen every block.  The
// consumer then adds the residual from the result region (tp_stage_c / _d).
//
// The O column-parallel projection's AllGather (H1) is fused the same way:
// its EPI_RESID epilogue (peer_mode 1) stores the rank's output slice into every rank's
// all-gather region (site 0's result region, [N][M][D/N]) and bumps every rank's site-0
// `done` counter; peer_wait on the network stream waits for all ranks' units.
//
// Flags and `done` counters reset themselves (a flag is cleared by its owner
// before the block's broadcast; `done` by its rank after the last block), which is
// safe because the next use of a site on any rank causally follows the completion
// of the current one on every rank.  Every wait is bounded: past
// the timeout the kernel records the event in the buffer's error word and exits
// (no hang), nf_comm_sym_status reports it.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

constexpr int PEER_BM = 128;            // rows of an owned block
constexpr int PEER_BN = 256;            // columns of an owned block
constexpr int PEER_SITES = 8;           // (O row-parallel, Down) x dense nano-batch (<= 4)
constexpr int64_t PEER_CTL_BYTES = 4096;  // buffer header: error word, timeouts

// Layout of one rank's symmetric buffer (identical on every rank of the group).
struct PeerGeom {
  int n = 1, rank = 0;    // group size, this rank
  int max_rows = 0, cols = 0;  // rows (tokens) and columns (d_model) a site can hold
  int maxb = 0, maxown = 0;    // 128x256 blocks of a full site, blocks one owner holds at most
  int64_t flags_off = 0;   // site-relative: done counter (u32) at 0, flags[maxown][n] at 256
  int64_t stage_off = 0;   // site-relative: partial staging [n][maxown][128][256] bf16
  int64_t result_off = 0;  // site-relative: result rows [max_rows][cols] bf16
  int64_t site_bytes = 0;
  int64_t total_bytes = 0;
  __host__ __device__ int64_t site(int s) const { return PEER_CTL_BYTES + (int64_t)s * site_bytes; }
};

PeerGeom peer_geom(int n, int rank, int max_rows, int cols);

// Owner-side reduce + broadcast of one site (grid: min(owned blocks, ctas) CTAs of 128 threads).
// bases: device array [n] of every rank's buffer base (this rank's mapping); M rows x geom.cols.
cudaError_t launch_peer_reduce(uint8_t* const* bases, const PeerGeom& g, int site, int M, int ctas,
                               long long timeout_ns, cudaStream_t st);

// Wait (one thread) until this rank's `done` counter of `site` reaches `expected` (the fused
// all-gather's producer units from every rank), then clear it.
cudaError_t launch_peer_wait(uint8_t* const* bases, const PeerGeom& g, int site, uint32_t expected, long long timeout_ns,
                             cudaStream_t st);

// Load every kernel of the library into the current context / a green context (see peer.cu).
cudaError_t preload_all_kernels();
cudaError_t preload_kernels_green(void* green_ctx);

}  // namespace nf
