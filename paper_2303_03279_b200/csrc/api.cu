// C ABI of csconn (include/csconn.h): plan lifetime, argument validation with
// the reference's error classes (core.py:17-22), kernel orchestration.
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace cs {
void run_spectra(const Plan& p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0, int kc,
                 cudaStream_t st);
void run_node_stats(const Plan& p, const int* slots, int K, int bin_lo, int nbb, cudaStream_t st);
void run_get_spectra(const Plan& p, const int* slots, int ns, int bin_lo, int nbins, void* dst,
                     cudaStream_t st);
void run_put_spectra(const Plan& p, const void* src, int n, int bin_lo, int nbins, int slot0, int taper, double w,
                     cudaStream_t st);
void run_pair_sums(const Plan& p, const int* slots, int K, int bin_lo, int nbb, const cs_sums* out, cudaStream_t st);
struct LagArgs;
int run_lag_family(Plan& p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                    int rb, int re, const cs_outputs* out, cudaStream_t st);
int run_coh_family(Plan& p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                    int rb, int re, const cs_outputs* out, cudaStream_t st);
}  // namespace cs

using cs::Plan;

static thread_local char g_err[512] = "";

void cs_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

struct cs_plan : Plan {};

namespace {
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
struct ProfState {
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
struct PhaseRec {
  ProfState* ps;
  cudaStream_t st;
  ProfRec r;
};
}  // namespace

cs::PhaseMark::PhaseMark(Plan& p, const char* name, cudaStream_t st) {
  p.launches += 1;
  if (!p.profiling) return;
  auto* pr = new PhaseRec{(ProfState*)p.prof, st, {}};
  pr->r.name = name;
  pr->r.a = pr->ps->get();
  pr->r.b = pr->ps->get();
  cudaEventRecord(pr->r.a, st);
  rec = pr;
}

cs::PhaseMark::~PhaseMark() {
  if (!rec) return;
  auto* pr = (PhaseRec*)rec;
  cudaEventRecord(pr->r.b, pr->st);
  pr->ps->recs.push_back(pr->r);
  delete pr;
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int cuda_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  cs_set_error("%s: %s", what, cudaGetErrorString(e));
  return CS_ECUDA;
}

bool is_pow2(double s) {
  int e;
  double m = std::frexp(s, &e);
  return m == 0.5;
}

// exp(-2 pi i m / n) with exact values on the axes
void twiddle(long m, long n, double* c, double* s) {
  m %= n;
  if (m == 0) { *c = 1.0; *s = 0.0; return; }
  if (2 * m == n) { *c = -1.0; *s = 0.0; return; }
  if (4 * m == n) { *c = 0.0; *s = -1.0; return; }
  if (4 * m == 3 * n) { *c = 0.0; *s = 1.0; return; }
  const long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)n;
  *c = (double)cosl(ang);
  *s = (double)(-sinl(ang));
}

}  // namespace

extern "C" {

const char* cs_last_error(void) { return g_err; }
const char* cs_version(void) { return "csconn 0.1 (sm_100a)"; }

int cs_num_row_tiles(int n_nodes) { return (n_nodes + cs::kTile - 1) / cs::kTile; }

int cs_row_tile_range(int n_nodes, int n_shards, int shard, int* rb, int* re, int64_t* p0,
                      int64_t* p1) {
  if (n_nodes < 1 || n_shards < 1 || shard < 0 || shard >= n_shards) {
    cs_set_error("cs_row_tile_range: bad arguments");
    return CS_EPARAM;
  }
  const int nt = cs_num_row_tiles(n_nodes);
  // balance by tile count: row I holds nt - I tiles
  const int64_t total = (int64_t)nt * (nt + 1) / 2;
  auto row_for = [&](int64_t target) {
    int64_t acc = 0;
    int r = 0;
    while (r < nt && acc + (nt - r) <= target) {
      acc += nt - r;
      ++r;
    }
    // round to the nearer boundary
    if (r < nt && target - acc > (acc + (nt - r)) - target) ++r;
    return r;
  };
  const int b = shard == 0 ? 0 : row_for(total * shard / n_shards);
  const int e = shard == n_shards - 1 ? nt : row_for(total * (shard + 1) / n_shards);
  *rb = b;
  *re = e;
  auto first_pair_of_row = [&](int64_t i) {
    if (i >= n_nodes) return (int64_t)n_nodes * (n_nodes - 1) / 2;
    return i * (n_nodes - 1) - i * (i - 1) / 2;
  };
  *p0 = first_pair_of_row((int64_t)b * cs::kTile);
  *p1 = first_pair_of_row((int64_t)e * cs::kTile);
  return CS_OK;
}

int cs_plan_create(cs_plan** out, int device, int N, int T, int nfft, int lo, int hi, int L,
                   const double* tapers, int slot_cap, double scale, unsigned flags) {
  if (!out) return CS_EPARAM;
  if (flags & ~CS_PLAN_WELCH) { cs_set_error("unknown plan flags 0x%x", flags); return CS_EPARAM; }
  int seg_stride = 0;
  if (flags & CS_PLAN_WELCH) {  // segments on the taper axis (spectral.py:100-111, 272-283)
    if (tapers || L != 1) { cs_set_error("welch mode takes no tapers"); return CS_EPARAM; }
    if (nfft >= 2 && T >= 2 * nfft) {
      L = T / nfft;
      seg_stride = nfft;
    }
  }
  *out = nullptr;
  if (nfft < 2) { cs_set_error("nfft must be >= 2, got %d", nfft); return CS_EPARAM; }
  if (N < 1) { cs_set_error("need at least one channel"); return CS_EPARAM; }
  if (T < 1) { cs_set_error("empty signal"); return CS_EPARAM; }
  const int nbins = nfft / 2 + 1;
  if (lo < 0 || hi < lo || hi >= nbins) {
    cs_set_error("invalid band bins [%d, %d] for %d bins", lo, hi, nbins);
    return CS_EPARAM;
  }
  if (L < 1 || (!tapers && L != 1 && !seg_stride)) { cs_set_error("bad taper count %d", L); return CS_EPARAM; }
  if (slot_cap < 1) { cs_set_error("slot_capacity must be >= 1"); return CS_EPARAM; }
  if (scale == 0.0) scale = 1.0;
  if (!(scale > 0.0) || !is_pow2(scale)) {
    cs_set_error("spectrum_scale must be a positive power of two");
    return CS_EPARAM;
  }
  DeviceGuard g(device);
  cs_plan* p = new cs_plan();
  p->device = device;
  p->N = N; p->ldn = N; p->T = T; p->nfft = nfft; p->lo = lo; p->hi = hi; p->nb = hi - lo + 1; p->L = L;
  p->T_eff = T < nfft ? T : nfft;
  p->seg_stride = seg_stride;
  p->slot_cap = slot_cap;
  p->scale = (float)scale;
  p->dc_local = (lo == 0) ? 0 : -1;
  p->nyq_local = (nfft % 2 == 0 && hi == nfft / 2) ? (nfft / 2 - lo) : -1;

  // taper x twiddle table (host fp64, long double angles)
  std::vector<double2> tw((size_t)L * p->nb * p->T_eff), ws((size_t)L * p->nb);
  for (int l = 0; l < L; ++l)
    for (int b = 0; b < p->nb; ++b) {
      long double sr = 0.0L, si = 0.0L;
      for (int t = 0; t < p->T_eff; ++t) {
        double c, s;
        twiddle((long)(lo + b) * t, nfft, &c, &s);
        const double w = tapers ? tapers[(size_t)l * p->T_eff + t] : 1.0;
        const double2 v = make_double2(w * c, w * s);
        tw[((size_t)l * p->nb + b) * p->T_eff + t] = v;
        sr += v.x;
        si += v.y;
      }
      ws[(size_t)l * p->nb + b] = make_double2((double)sr, (double)si);
    }
  // FFT path: power-of-two nfft and a band for which ~5 M log2 M flops beat 4 T_eff nb
  {
    const bool pow2 = nfft >= 8 && (nfft & (nfft - 1)) == 0;
    const int M = nfft / 2;
    int lg = 0;
    while ((1 << lg) < M) ++lg;
    const char* force = getenv("CSCONN_SPECTRA");
    p->use_fft = pow2 && (force ? force[0] == 'f' : (5.0 * M * lg + 16.0 * M < 4.0 * p->T_eff * p->nb));
  }
  const int64_t P = (int64_t)N * (N - 1) / 2;
  int64_t cap = P * p->nb / 64;
  if (cap < (1 << 16)) cap = 1 << 16;
  if (cap > (1 << 24)) cap = 1 << 24;
  if (const char* fc = getenv("CSCONN_FLAG_CAP")) cap = atol(fc) > 0 ? atol(fc) : 1;  // test override (overflow path)
  p->flag_cap = (int)cap;
  const size_t ring = (size_t)slot_cap * L * p->nb * N;
  bool ok = cudaMalloc(&p->tww, tw.size() * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&p->wsum, ws.size() * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&p->X64, ring * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&p->X32, ring * sizeof(float2)) == cudaSuccess &&
            cudaMalloc(&p->psd, (size_t)p->nb * N * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&p->mag, (size_t)p->nb * N * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&p->nscale, (size_t)p->nb * N * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&p->flags, (size_t)p->flag_cap * sizeof(int4)) == cudaSuccess &&
            cudaMalloc(&p->counters, 4 * sizeof(int)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    cs_set_error("device allocation failed (spectrum ring %zu bytes)", ring * 24);
    cs_plan_destroy(p);
    return CS_ENOMEM;
  }
  cudaMemcpy(p->tww, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemcpy(p->wsum, ws.data(), ws.size() * sizeof(double2), cudaMemcpyHostToDevice);
  // tensor-core DFT: B fragments of mma.m8n8k4.f64 in lane order; columns 2b, 2b+1 =
  // taper x twiddle (Re, Im) of bin b, column 2 nb = 1 (untapered sample sum)
  if (!p->use_fft && 2 * p->nb + 1 <= 24 && !(getenv("CSCONN_DFT") && getenv("CSCONN_DFT")[0] == 'f')) {
    const int NT = (2 * p->nb + 1 + 7) / 8, nks = (p->T_eff + 3) / 4;
    std::vector<double> tf((size_t)L * nks * NT * 32, 0.0);
    for (int l = 0; l < L; ++l)
      for (int kk = 0; kk < nks; ++kk)
        for (int nt = 0; nt < NT; ++nt)
          for (int ln = 0; ln < 32; ++ln) {
            const int t = 4 * kk + (ln & 3), col = nt * 8 + (ln >> 2);
            double v = 0.0;
            if (t < p->T_eff) {
              if (col < 2 * p->nb) {
                const double2 w = tw[((size_t)l * p->nb + col / 2) * p->T_eff + t];
                v = (col & 1) ? w.y : w.x;
              } else if (col == 2 * p->nb) {
                v = 1.0;
              }
            }
            tf[(((size_t)l * nks + kk) * NT + nt) * 32 + ln] = v;
          }
    if (cudaMalloc(&p->dft_tf, tf.size() * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      p->dft_tf = nullptr;  // the DFMA kernel needs no extra table
    } else {
      cudaMemcpy(p->dft_tf, tf.data(), tf.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  if (p->use_fft) {
    const int M = nfft / 2;
    std::vector<double2> ft(M / 2 > 0 ? M / 2 : 1), pt(M + 1);
    for (int j = 0; j < M / 2; ++j) {
      double c, s;
      twiddle(j, M, &c, &s);
      ft[j] = make_double2(c, s);
    }
    for (int k = 0; k <= M; ++k) {
      double c, s;
      twiddle(k, nfft, &c, &s);
      pt[k] = make_double2(c, s);
    }
    bool ok2 = cudaMalloc(&p->fft_tw, ft.size() * sizeof(double2)) == cudaSuccess &&
               cudaMalloc(&p->post_tw, pt.size() * sizeof(double2)) == cudaSuccess;
    if (tapers) ok2 = ok2 && cudaMalloc(&p->taper, (size_t)L * p->T_eff * sizeof(double)) == cudaSuccess;
    if (!ok2) {
      cudaGetLastError();
      cs_set_error("device allocation failed (FFT tables)");
      cs_plan_destroy(p);
      return CS_ENOMEM;
    }
    cudaMemcpy(p->fft_tw, ft.data(), ft.size() * sizeof(double2), cudaMemcpyHostToDevice);
    cudaMemcpy(p->post_tw, pt.data(), pt.size() * sizeof(double2), cudaMemcpyHostToDevice);
    if ((M == 256 || M == 512) && !(getenv("CSCONN_FFT") && getenv("CSCONN_FFT")[0] == 'r')) {
      const int A = M / 32;  // four-step tables: W_M^{b k_a} [k_a][b], then W_32^j
      std::vector<double2> t4((size_t)A * 32 + 32);
      for (int ka = 0; ka < A; ++ka)
        for (int b = 0; b < 32; ++b) {
          double c, s;
          twiddle((long)b * ka, M, &c, &s);
          t4[(size_t)ka * 32 + b] = make_double2(c, s);
        }
      for (int j = 0; j < 32; ++j) {
        double c, s;
        twiddle(j, 32, &c, &s);
        t4[(size_t)A * 32 + j] = make_double2(c, s);
      }
      if (cudaMalloc(&p->fft4_tw, t4.size() * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        cs_set_error("device allocation failed (FFT tables)");
        cs_plan_destroy(p);
        return CS_ENOMEM;
      }
      cudaMemcpy(p->fft4_tw, t4.data(), t4.size() * sizeof(double2), cudaMemcpyHostToDevice);
    }
    if (tapers) cudaMemcpy(p->taper, tapers, (size_t)L * p->T_eff * sizeof(double), cudaMemcpyHostToDevice);
  }
  cudaMemset(p->X64, 0, ring * sizeof(double2));
  cudaMemset(p->X32, 0, ring * sizeof(float2));
  cudaMemset(p->counters, 0, 4 * sizeof(int));
  if (cudaGetLastError() != cudaSuccess) {
    cs_plan_destroy(p);
    return cuda_fail("cs_plan_create");
  }
  *out = p;
  return CS_OK;
}

int cs_plan_destroy(cs_plan* p) {
  if (!p) return CS_OK;
  DeviceGuard g(p->device);
  cudaFree(p->tww); cudaFree(p->wsum); cudaFree(p->taper); cudaFree(p->fft_tw); cudaFree(p->post_tw); cudaFree(p->fft4_tw); cudaFree(p->dft_tf); cudaFree(p->X64); cudaFree(p->X32); cudaFree(p->psd); cudaFree(p->mag); cudaFree(p->nscale);
  if (p->tc_ops) cudaFree(p->tc_ops);
  for (auto& e : p->tc_tiles)
    if (e.ptr) cudaFree(e.ptr);
  if (p->lag_ops) cudaFree(p->lag_ops);
  cudaFree(p->flags); cudaFree(p->counters);
  if (p->peer_x64) cudaFree(p->peer_x64);
  for (void* m : p->ipc_opened) cudaIpcCloseMemHandle(m);
  if (p->recs) cudaFree(p->recs);
  if (p->prof) {
    auto* ps = (ProfState*)p->prof;
    for (auto& r : ps->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ps->pool) cudaEventDestroy(e);
    delete ps;
  }
  delete p;
  return CS_OK;
}

int cs_spectra(cs_plan* p, const void* x, int dtype, int64_t ts, int64_t ns, int slot0, int kc,
               void* stream) {
  if (!p || !x) { cs_set_error("cs_spectra: null argument"); return CS_EPARAM; }
  if (dtype != CS_F32 && dtype != CS_F64) { cs_set_error("unknown dtype %d", dtype); return CS_EPARAM; }
  if (kc < 0 || slot0 < 0) { cs_set_error("cs_spectra: bad trial range"); return CS_EPARAM; }
  if (kc == 0) return CS_OK;
  DeviceGuard g(p->device);
  {
    cs::PhaseMark ph(*p, "spectra", (cudaStream_t)stream);
    // trials x tapers ride on a grid dimension (<= 65535): chunk long calls
    const int step = 65535 / p->L;
    const size_t esz = dtype == CS_F64 ? 8 : 4;
    for (int c0 = 0; c0 < kc; c0 += step)
      cs::run_spectra(*p, (const char*)x + (size_t)c0 * ts * esz, dtype, ts, ns, (slot0 + c0) % p->slot_cap,
                      kc - c0 < step ? kc - c0 : step, (cudaStream_t)stream);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cs_spectra");
  p->fft_calls += (int64_t)kc * p->N * p->L;
  return CS_OK;
}

int cs_pair_metrics(cs_plan* p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                    int rb, int re, const cs_outputs* out, void* stream) {
  return cs_pair_metrics_ex(p, slots, K, mask, bin_lo, nbb, rb, re, out, 0u, stream);
}

int cs_pair_metrics_ex(cs_plan* p, const int* slots, int K, unsigned mask, int bin_lo, int nbb,
                       int rb, int re, const cs_outputs* out, unsigned flags, void* stream) {
  if (!p || !out) { cs_set_error("cs_pair_metrics: null argument"); return CS_EPARAM; }
  if (flags & ~CS_PM_REUSE_PREP) { cs_set_error("unknown pair-metrics flags 0x%x", flags); return CS_EPARAM; }
  if (mask == 0 || (mask >> CS_NUM_METRICS)) { cs_set_error("bad metric mask 0x%x", mask); return CS_EPARAM; }
  if (K < 1) { cs_set_error("no trials accumulated"); return CS_EDEGENERATE; }
  if ((mask & CS_USPLI) && K < 2) { cs_set_error("USPLI needs at least 2 trials"); return CS_EDEGENERATE; }
  if (bin_lo < 0 || nbb < 1 || bin_lo + nbb > p->nb) {
    cs_set_error("bins [%d, %d) outside the plan's %d bins", bin_lo, bin_lo + nbb, p->nb);
    return CS_EPARAM;
  }
  const int nt = cs_num_row_tiles(p->N);
  if (re < 0) re = nt;
  if (rb < 0 || rb > re || re > nt) { cs_set_error("bad row tile range [%d, %d)", rb, re); return CS_EPARAM; }
  if (p->N < 2 || rb == re) return CS_OK;
  DeviceGuard g(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  Plan::PrepKey key;
  key.slots = slots; key.K = K; key.bin_lo = bin_lo; key.nbb = nbb; key.mask = mask;
  const bool reuse = (flags & CS_PM_REUSE_PREP) != 0;
  if (reuse && !(p->prep_valid && p->prep_key == key)) {
    cs_set_error("CS_PM_REUSE_PREP: the previous call prepared other slots, bins or metrics");
    return CS_EPARAM;
  }
  p->reuse_prep = reuse;
  p->prep_valid = false;
  if (!reuse) {
    cs::PhaseMark ph(*p, "node_stats", st);
    cs::run_node_stats(*p, slots, K, bin_lo, nbb, st);
  }
  // only the requested metrics' buffers are ever written
  cs_outputs o = *out;
  for (int m = 0; m < CS_NUM_METRICS; ++m)
    if (!(mask & (1u << m))) o.bins[m] = o.band[m] = nullptr;
  // tensor-core family (COHY, COH, PLV; IMAGCOHY when no sign-based metric is asked),
  // then the phase-lag family
  p->imag_handoff = false;
  const int rc1 = cs::run_coh_family(*p, slots, K, mask, bin_lo, nbb, rb, re, &o, st);
  const int rc2 = rc1 < 0 ? -1 : cs::run_lag_family(*p, slots, K, mask, bin_lo, nbb, rb, re, &o, st);
  p->reuse_prep = false;
  if (rc1 < 0 || rc2 < 0) return CS_EPARAM;
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cs_pair_metrics");
  p->prep_key = key;
  p->prep_valid = true;
  return CS_OK;
}

int cs_get_spectra(cs_plan* p, const int* slots, int ns, int bin_lo, int nbins, void* dst,
                   void* stream) {
  if (!p || !slots || !dst) { cs_set_error("cs_get_spectra: null argument"); return CS_EPARAM; }
  if (bin_lo < 0 || nbins < 1 || bin_lo + nbins > p->nb) { cs_set_error("cs_get_spectra: bad bins"); return CS_EPARAM; }
  if (ns <= 0) return CS_OK;
  DeviceGuard g(p->device);
  for (int c0 = 0; c0 < ns; c0 += 65535)  // trials ride on grid.y
    cs::run_get_spectra(*p, slots + c0, ns - c0 < 65535 ? ns - c0 : 65535, bin_lo, nbins,
                        (double2*)dst + (size_t)c0 * p->N * nbins, (cudaStream_t)stream);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cs_get_spectra");
  return CS_OK;
}

int cs_put_spectra(cs_plan* p, const void* src, int n, int bin_lo, int nbins, int slot0, void* stream) {
  return cs_put_taper_spectra(p, src, n, bin_lo, nbins, slot0, 0, 1.0, stream);
}

int cs_put_taper_spectra(cs_plan* p, const void* src, int n, int bin_lo, int nbins, int slot0, int taper,
                         double w, void* stream) {
  if (!p || !src) { cs_set_error("cs_put_spectra: null argument"); return CS_EPARAM; }
  if (taper < 0 || taper >= p->L) { cs_set_error("cs_put_spectra: taper %d outside [0, %d)", taper, p->L); return CS_EPARAM; }
  if (bin_lo < 0 || nbins < 1 || bin_lo + nbins > p->nb || slot0 < 0) {
    cs_set_error("cs_put_spectra: bad bins/slot");
    return CS_EPARAM;
  }
  if (n <= 0) return CS_OK;
  DeviceGuard g(p->device);
  p->spectra_put = true;  // arbitrary spectra: no exactly-real DC / Nyquist shortcut from now on
  {
    cs::PhaseMark ph(*p, "put_spectra", (cudaStream_t)stream);
    for (int c0 = 0; c0 < n; c0 += 65535)  // trials ride on grid.y
      cs::run_put_spectra(*p, (const double2*)src + (size_t)c0 * p->N * nbins, n - c0 < 65535 ? n - c0 : 65535,
                          bin_lo, nbins, (slot0 + c0) % p->slot_cap, taper, w, (cudaStream_t)stream);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cs_put_spectra");
  return CS_OK;
}

int cs_last_fallback_count(cs_plan* p, void* stream, int64_t* n) {
  int64_t rec = 0;
  return cs_last_guard_stats(p, stream, n, &rec);
}

int cs_last_guard_stats(cs_plan* p, void* stream, int64_t* n, int64_t* records) {
  if (!p || !n || !records) return CS_EPARAM;
  DeviceGuard g(p->device);
  int h[3] = {0, 0, 0};
  if (cudaMemcpyAsync(h, p->counters, 3 * sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream) !=
          cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
    return cuda_fail("cs_last_guard_stats");
  *n = h[0];
  *records = h[2];
  return CS_OK;
}

int cs_plan_set_profiling(cs_plan* p, int on) {
  if (!p) return CS_EPARAM;
  if (!p->prof) p->prof = new ProfState();
  p->profiling = on != 0;
  return CS_OK;
}

int cs_profile_read(cs_plan* p, char* buf, int len) {
  if (!p || !buf || len < 1) return CS_EPARAM;
  buf[0] = 0;
  if (!p->prof) return CS_OK;
  DeviceGuard g(p->device);
  auto* ps = (ProfState*)p->prof;
  struct Acc { const char* name; double ms; int n; };
  std::vector<Acc> acc;
  for (auto& r : ps->recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& a : acc)
      if (!strcmp(a.name, r.name)) { a.ms += ms; a.n++; found = true; }
    if (!found) acc.push_back({r.name, (double)ms, 1});
    ps->pool.push_back(r.a);
    ps->pool.push_back(r.b);
  }
  ps->recs.clear();
  int off = 0;
  for (auto& a : acc) off += snprintf(buf + off, len > off ? len - off : 0, "%s:%.6f:%d;", a.name, a.ms, a.n);
  return CS_OK;
}

int64_t cs_launch_count(const cs_plan* p) { return p ? p->launches : 0; }

int cs_ring_view(cs_plan* p, void** x64, void** x32, int64_t* n_elems) {
  if (!p) return CS_EPARAM;
  *x64 = p->X64;
  *x32 = p->X32;
  *n_elems = (int64_t)p->slot_cap * p->L * p->nb * p->N;
  return CS_OK;
}

int64_t cs_fft_call_count(const cs_plan* p) { return p ? p->fft_calls : 0; }
int cs_last_imag_handoff(const cs_plan* p) { return !p ? 0 : p->imag_handoff ? 1 : 0; }

int cs_plan_k1_kind(const cs_plan* p) {
  if (!p) return -1;
  if (p->use_fft) return (p->fft4_tw && (p->nfft == 512 || p->nfft == 1024)) ? 2 : 3;
  return p->dft_tf ? 1 : 0;
}
void cs_reset_fft_call_count(cs_plan* p) { if (p) p->fft_calls = 0; }

int cs_pair_sums(cs_plan* p, const int* slots, int K, int bin_lo, int nbb, const cs_sums* out, void* stream) {
  if (!p || !out || (!slots && K > 0)) { cs_set_error("cs_pair_sums: null argument"); return CS_EPARAM; }
  if (K < 0) { cs_set_error("cs_pair_sums: negative trial count"); return CS_EPARAM; }
  if (bin_lo < 0 || nbb < 1 || bin_lo + nbb > p->nb) {
    cs_set_error("bins [%d, %d) outside the plan's %d bins", bin_lo, bin_lo + nbb, p->nb);
    return CS_EPARAM;
  }
  if (out->pair_base < 0 || out->pair_stride < 0) { cs_set_error("cs_pair_sums: bad pair range"); return CS_EPARAM; }
  DeviceGuard g(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  {
    cs::PhaseMark ph(*p, "pair_sums", st);
    cs::run_pair_sums(*p, slots, K, bin_lo, nbb, out, st);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cs_pair_sums");
  return CS_OK;
}

}  // extern "C"
