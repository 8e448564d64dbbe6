// Multi-GPU exchange of the spectrum ring over NVLink peer memory.
//
// Every rank holds a plan over all N nodes.  Rank r runs K1 for its node block only
// (cs_spectra_nodes: the block's columns of its own ring), then pushes that block of
// the fp32 ring into every peer's ring with strided copy-engine copies
// (cs_ring_push: one cudaMemcpy2DAsync per peer over the IPC-mapped peer ring, no
// staging buffer, no SM time).  The fp64 ring is not exchanged: only the exact-sign
// fallback reads it (~5e-4 of the (pair, bin) entries), and it loads a remote node's
// fp64 spectra straight from the owning rank's ring through the attached peer
// pointer table (P2P loads over NVLink).
//
// The reference has no multi-process path: this is the B200 layout of
// the partition in north_star ("node spectra all-gathered over NVLink, only the
// pair-tile results return").
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {
struct DevG {
  int prev = -1;
  explicit DevG(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevG() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
int fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  cs_set_error("%s: %s", what, cudaGetErrorString(e));
  return CS_ECUDA;
}
}  // namespace

struct cs_plan;
namespace cs {
void run_spectra(const Plan& p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0, int kc,
                 cudaStream_t st);
}

extern "C" {

int cs_spectra_nodes(cs_plan* plan, const void* x, int dtype, int64_t ts, int64_t ns, int node0, int n_nodes,
                     int slot0, int kc, void* stream) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!p || !x) { cs_set_error("cs_spectra_nodes: null argument"); return CS_EPARAM; }
  if (dtype != CS_F32 && dtype != CS_F64) { cs_set_error("unknown dtype %d", dtype); return CS_EPARAM; }
  if (node0 < 0 || n_nodes < 0 || node0 + n_nodes > p->N) {
    cs_set_error("node range [%d, %d) outside the plan's %d nodes", node0, node0 + n_nodes, p->N);
    return CS_EPARAM;
  }
  if (kc < 0 || slot0 < 0) { cs_set_error("cs_spectra_nodes: bad trial range"); return CS_EPARAM; }
  if (kc == 0 || n_nodes == 0) return CS_OK;
  DevG g(p->device);
  // a view of the plan over the node range: same ring rows (ldn), columns from node0
  cs::Plan v = *p;
  v.N = n_nodes;
  v.X64 = p->X64 + node0;
  v.X32 = p->X32 + node0;
  {
    cs::PhaseMark ph(*p, "spectra", (cudaStream_t)stream);
    const int step = 65535 / p->L;
    const size_t esz = dtype == CS_F64 ? 8 : 4;
    for (int c0 = 0; c0 < kc; c0 += step)
      cs::run_spectra(v, (const char*)x + (size_t)c0 * ts * esz, dtype, ts, ns, (slot0 + c0) % p->slot_cap,
                      kc - c0 < step ? kc - c0 : step, (cudaStream_t)stream);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return fail("cs_spectra_nodes");
  p->fft_calls += (int64_t)kc * n_nodes * p->L;
  return CS_OK;
}

int cs_ring_export(cs_plan* plan, cs_ring_handle* out) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!p || !out) { cs_set_error("cs_ring_export: null argument"); return CS_EPARAM; }
  DevG g(p->device);
  memset(out, 0, sizeof(*out));
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(out->x64), "IPC handle size");
  if (cudaIpcGetMemHandle((cudaIpcMemHandle_t*)out->x64, p->X64) != cudaSuccess ||
      cudaIpcGetMemHandle((cudaIpcMemHandle_t*)out->x32, p->X32) != cudaSuccess)
    return fail("cs_ring_export");
  out->n_nodes = p->N;
  out->slot_capacity = p->slot_cap;
  out->n_tapers = p->L;
  out->n_bins = p->nb;
  return CS_OK;
}

static int attach(cs::Plan* p, void* const* x64, void* const* x32, int n_ranks, int self, int node_block) {
  if (n_ranks < 1 || self < 0 || self >= n_ranks || node_block < 1 ||
      (int64_t)node_block * n_ranks < p->N) {
    cs_set_error("cs_ring_attach: bad rank layout (%d ranks, self %d, node block %d, %d nodes)", n_ranks, self,
                 node_block, p->N);
    return CS_EPARAM;
  }
  if (p->peer_x64) cudaFree(p->peer_x64);
  p->peer_x64 = nullptr;
  if (cudaMalloc(&p->peer_x64, n_ranks * sizeof(double2*)) != cudaSuccess) return fail("cs_ring_attach");
  std::vector<double2*> t(n_ranks);
  for (int r = 0; r < n_ranks; ++r) t[r] = r == self ? p->X64 : (double2*)x64[r];
  cudaMemcpy(p->peer_x64, t.data(), n_ranks * sizeof(double2*), cudaMemcpyHostToDevice);
  p->peers32.assign(n_ranks, nullptr);
  for (int r = 0; r < n_ranks; ++r) p->peers32[r] = r == self ? nullptr : (float2*)x32[r];
  p->n_ranks = n_ranks;
  p->rank = self;
  p->node_block = node_block;
  return cudaGetLastError() == cudaSuccess ? CS_OK : fail("cs_ring_attach");
}

int cs_ring_attach(cs_plan* plan, const cs_ring_handle* peers, int n_ranks, int self, int node_block) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!p || !peers) { cs_set_error("cs_ring_attach: null argument"); return CS_EPARAM; }
  DevG g(p->device);
  std::vector<void*> x64(n_ranks, nullptr), x32(n_ranks, nullptr);
  for (int r = 0; r < n_ranks; ++r) {
    const cs_ring_handle& h = peers[r];
    if (h.n_nodes != p->N || h.slot_capacity != p->slot_cap || h.n_tapers != p->L || h.n_bins != p->nb) {
      cs_set_error("cs_ring_attach: rank %d's ring has another geometry", r);
      return CS_EPARAM;
    }
    if (r == self) continue;
    cudaIpcMemHandle_t a, b;
    memcpy(&a, h.x64, sizeof(a));
    memcpy(&b, h.x32, sizeof(b));
    if (cudaIpcOpenMemHandle(&x64[r], a, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&x32[r], b, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return fail("cs_ring_attach (cudaIpcOpenMemHandle)");
    p->ipc_opened.push_back(x64[r]);
    p->ipc_opened.push_back(x32[r]);
  }
  return attach(p, x64.data(), x32.data(), n_ranks, self, node_block);
}

int cs_ring_attach_ptrs(cs_plan* plan, void* const* x64, void* const* x32, int n_ranks, int self, int node_block) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!p || !x64 || !x32) { cs_set_error("cs_ring_attach_ptrs: null argument"); return CS_EPARAM; }
  DevG g(p->device);
  return attach(p, x64, x32, n_ranks, self, node_block);
}

int cs_ring_push(cs_plan* plan, int node0, int n_nodes, int slot0, int kc, void* stream) {
  cs::Plan* p = (cs::Plan*)plan;
  if (!p) { cs_set_error("cs_ring_push: null plan"); return CS_EPARAM; }
  if (p->n_ranks < 1) { cs_set_error("cs_ring_push: no peers attached"); return CS_EPARAM; }
  if (node0 < 0 || n_nodes < 0 || node0 + n_nodes > p->N || kc < 0 || kc > p->slot_cap || slot0 < 0) {
    cs_set_error("cs_ring_push: bad node / slot range");
    return CS_EPARAM;
  }
  if (n_nodes == 0 || kc == 0) return CS_OK;
  DevG g(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t rows_per_slot = (size_t)p->L * p->nb, pitch = (size_t)p->ldn * sizeof(float2);
  int s = slot0 % p->slot_cap, left = kc;
  while (left > 0) {  // slot runs that do not wrap
    const int run = left < p->slot_cap - s ? left : p->slot_cap - s;
    const size_t off = (size_t)s * rows_per_slot * p->ldn + node0;
    for (int r = 0; r < p->n_ranks; ++r) {
      if (!p->peers32[r]) continue;
      if (cudaMemcpy2DAsync(p->peers32[r] + off, pitch, p->X32 + off, pitch, (size_t)n_nodes * sizeof(float2),
                            run * rows_per_slot, cudaMemcpyDefault, st) != cudaSuccess)
        return fail("cs_ring_push");
    }
    left -= run;
    s = 0;
  }
  return CS_OK;
}

}  // extern "C"
