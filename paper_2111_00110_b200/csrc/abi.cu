// extern "C" entry points (include/fc2t2_b200.h) and the engine handle.
//
// The engine owns the device copy of the M2L tables of one
// Engine(kernel, levels) (reference expansion.py:157-177): fp32 PPxPP
// matrices B[n][k] = A_o[k][n] for every *active* offset (the interaction
// lists, kernel.py:275) and, per level, the list of (offset, slot) entries
// grouped by target parity class.  For a parity stencil level
// (reference expansion.py:236, :246-249) class (px, py, pz) sees -3 only on
// odd axes and +3 only on even axes; the coarsest level and the near table
// have one class.  At the finest level the near table is merged into every
// class list so one M2L pass applies far + near.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/fc2t2_b200.h"
#include "common.cuh"
#include "kernels.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FC2T2_OK;
  return fail(FC2T2_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

struct HostTable {
  bool set = false;
  std::vector<int64_t> offsets;  // K*3
  std::vector<uint8_t> active;   // K
  std::vector<double> coeffs;    // K*P*P
};

struct Plan {
  int stride = 1, ncls = 1;
  std::vector<int4> entries;
  std::vector<int> cls_start;
  int4* d_entries = nullptr;
  int* d_cls_start = nullptr;
  int max_list = 0;
  // tcgen05 form (parity levels): dense split tables, see build_tc_table
  bool tc = false;
  std::vector<uint8_t> tcb;
  std::vector<float> rk, s_inv;
  uint8_t* d_tcb = nullptr;
  float* d_rk = nullptr;
  float* d_sinv = nullptr;
};

}  // namespace

// ------------------------------------------------------------ profiling ---
namespace fc2t2 {
namespace {
std::atomic<long long> g_launches{0};
bool g_prof = false;
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;
const char* g_pending = nullptr;
cudaEvent_t g_pending_ev;

cudaEvent_t next_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}
}  // namespace

// FC2T2_DEBUG_ERRORS=1: report a launch that fails, or a CUDA error left
// pending by an earlier runtime call, naming the kernel (stderr)
const char* g_last_name = "(none)";
bool debug_errors() {
  static const bool v = [] {
    const char* e = std::getenv("FC2T2_DEBUG_ERRORS");
    return e && e[0] == '1';
  }();
  return v;
}

void prof_begin(const char* name, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (debug_errors()) {
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess)
      std::fprintf(stderr, "fc2t2: pending CUDA error before launch %s (previous launch %s): %s\n",
                   name, g_last_name, cudaGetErrorString(e));
    g_last_name = name;
  }
  if (!g_prof) return;
  g_pending_ev = next_event();
  cudaEventRecord(g_pending_ev, s);
  g_pending = name;
}

void prof_end(cudaStream_t s) {
  if (debug_errors()) {
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess)
      std::fprintf(stderr, "fc2t2: launch %s: %s\n", g_last_name, cudaGetErrorString(e));
  }
  if (!g_prof || !g_pending) return;
  cudaEvent_t b = next_event();
  cudaEventRecord(b, s);
  g_recs.push_back({g_pending, g_pending_ev, b});
  g_pending = nullptr;
}
}  // namespace fc2t2

struct fc2t2_engine {
  int rho = 0, levels = 0, P = 0, PP = 0;
  std::map<int, HostTable> far;
  HostTable near;
  bool uploaded = false;
  float* d_coef = nullptr;
  // plans[level][table]
  std::map<int, std::map<int, Plan>> plans;
  // fork/join for fc2t2_expand: the finest-level M2L runs on `side` while the
  // M2M chain and the coarse levels run on the caller's stream
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // coarse levels: every level's M2L on its own stream (cs[l & 1]) as soon as
  // its M grid exists (ev_m[l]); the L2L chain waits for each (ev_c[l])
  cudaStream_t cs[2] = {nullptr, nullptr};
  // the M2M chain of an overlapped cascade: high priority like cs[], so the
  // coarse chain's few CTAs are placed ahead of the finest level's many
  cudaStream_t up = nullptr;
  cudaEvent_t ev_m[10] = {}, ev_c[10] = {};
  // separable finest M2L (m2l_sep.cu): per-axis factors, [out][in] float64
  bool sep = false;
  bool sep_fuse_l2l = true;  // fc2t2_engine_set_sep_fusion
  std::vector<double> sep_pre, sep_post, sep_conv;
  // separable far tables of coarse levels: level -> {pre, post, conv}
  // (fc2t2_engine_set_separable_far)
  std::map<int, std::vector<double>> sep_far;
};

namespace {

constexpr int kCoarsest = 2;

// host round-to-nearest-even to fp16; returns the bits and the exact value
uint16_t half_rn(double v, double* val) {
  const uint16_t sign = v < 0 ? 0x8000 : 0;
  const double a = std::fabs(v);
  uint16_t bits = 0;
  double r = 0.0;
  if (a > 0.0) {
    int ex;
    std::frexp(a, &ex);
    int E = ex - 1;  // a in [2^E, 2^(E+1))
    if (E < -14) {
      const double q = std::nearbyint(std::ldexp(a, 24));
      bits = (uint16_t)q;
      r = std::ldexp(q, -24);
    } else {
      double q = std::nearbyint(std::ldexp(a, 10 - E));
      if (q >= 2048.0) {
        q = 1024.0;
        ++E;
      }
      if (E > 15) {  // clamp (the scaling keeps |x| <= 2^13)
        E = 15;
        q = 2047.0;
      }
      bits = (uint16_t)(((E + 15) << 10) | ((int)q - 1024));
      r = std::ldexp(q, E - 10);
    }
  }
  *val = sign ? -r : r;
  return (uint16_t)(sign | bits);
}

// Dense tcgen05 tables of one parity plan (m2l_tc.cu): for class group cg
// (target classes cg*CLS + ci), source class sigma, shift slot
// s = (slot/9 - 1, slot/3%3 - 1, slot%3 - 1) and K step, the B operand rows
// are the CLS tables A_delta, delta = 2 s + sigma - pi (the sum of the plan's
// entries with that offset for class pi; zero if none), split in float64 into
// hi and lo parts.  Row order: even sigma [lo(class 0..) | hi(class 0..)], odd
// sigma [hi | lo]; K-major no-swizzle [kchunk][row][16 B].  B' = A s_n / r_k,
// hi = rn_f16(B'), lo = rn_f16((B' - hi) 2^11), with s_n = (h/2)^|n|/n! at the
// plan's level and r_k a power of two with max_{slot,n} |B'| <= 2^13
// (returned in rk, NC entries; s_inv = 1/s_n).
void build_tc_table(const std::vector<std::vector<int4>>& lists,
                    const std::vector<const double*>& slot_src, int P, int PP, int rho, int level,
                    Plan& plan) {
  int CLS, NC, KS, BSLOT, FL, TILES;
  if (fc2t2::tc_geometry(rho, &CLS, &NC, &KS, &BSLOT, &FL, &TILES) != 0) return;
  const bool SB = FL & 1, MERGE = FL & 2;
  const int W = CLS * NC, R = 2 * W, NCG = 8 / CLS;
  constexpr int KI = 16, ESZ = 2;
  std::vector<double> sn(P, 1.0);
  fc2t2::tc_moment_scales(rho, level, sn.data());
  plan.s_inv.assign(PP, 0.f);
  for (int n = 0; n < P; ++n) plan.s_inv[n] = (float)(1.0 / sn[n]);
  // per output column k: power of two r_k with max |A[k][n] s_n| / r_k <= 2^13
  std::vector<double> rk(NC, 1.0);
  {
    std::vector<double> mx(P, 0.0);
    for (const auto& l : lists)
      for (const int4& e : l) {
        const double* A = slot_src[e.w];
        for (int k = 0; k < P; ++k)
          for (int n = 0; n < P; ++n) mx[k] = std::max(mx[k], std::fabs(A[(size_t)k * P + n] * sn[n]));
      }
    for (int k = 0; k < P; ++k)
      if (mx[k] > 0.0) {
        int ex;
        std::frexp(mx[k], &ex);            // mx < 2^ex
        rk[k] = std::ldexp(1.0, ex - 13);
      }
  }
  plan.rk.assign(NC, 1.f);
  for (int k = 0; k < NC; ++k) plan.rk[k] = (float)rk[k];
  plan.tcb.assign((size_t)NCG * 8 * KS * 27 * BSLOT, 0);
  std::vector<double> A((size_t)P * P);
  for (int cg = 0; cg < NCG; ++cg)
    for (int sg = 0; sg < 8; ++sg) {
      const int sig[3] = {(sg >> 2) & 1, (sg >> 1) & 1, sg & 1};
      for (int slot = 0; slot < 27; ++slot) {
        const int sh[3] = {slot / 9 - 1, (slot / 3) % 3 - 1, slot % 3 - 1};
        for (int ci = 0; ci < CLS; ++ci) {
          const int c = cg * CLS + ci;
          const int pi[3] = {(c >> 2) & 1, (c >> 1) & 1, c & 1};
          int dl[3];
          for (int a = 0; a < 3; ++a) dl[a] = 2 * sh[a] + sig[a] - pi[a];
          std::fill(A.begin(), A.end(), 0.0);
          bool any = false;
          for (const int4& e : lists[c])
            if (e.x == dl[0] && e.y == dl[1] && e.z == dl[2]) {
              const double* src = slot_src[e.w];
              for (size_t i = 0; i < A.size(); ++i) A[i] += src[i];
              any = true;
            }
          if (!any) continue;
          const bool odd = (sg & 1) && !SB;   // single-buffered kernels keep [lo | hi]
          // rows [lo | hi] (even) or [hi | lo] (odd), 2W per slot
          const int f = ci * NC;                     // flattened (class, k) base
          for (int ks = 0; ks < KS; ++ks) {
              const int hi_row = odd ? f : W + f;
              const int lo_row = odd ? W + f : f;
              uint8_t* st = plan.tcb.data() +
                            ((((size_t)cg * 8 + sg) * KS + ks) * 27 + slot) * BSLOT;
              const bool merged = MERGE && ks == KS - 1;
              for (int kc = 0; kc < 2; ++kc)
                for (int k = 0; k < P; ++k)
                  for (int fi = 0; fi < KI / 2; ++fi) {
                    const int n = KI * ks + (merged ? 0 : (KI / 2) * kc) + fi;
                    if (n >= P) continue;
                    const double a = A[(size_t)k * P + n];
                    uint8_t hb[2], lb[2];
                    const double b = a * sn[n] / rk[k];
                    double hv, lv;
                    const uint16_t h16 = half_rn(b, &hv);
                    const uint16_t l16 = half_rn((b - hv) * 2048.0, &lv);
                    std::memcpy(hb, &h16, 2);
                    std::memcpy(lb, &l16, 2);
                    auto put = [&](int row, const uint8_t* v) {
                      std::memcpy(st + ((size_t)kc * R + row) * 16 + fi * ESZ, v, ESZ);
                    };
                    if (merged && kc == 1) {
                      // chunk 1 multiplies the A_lo chunk: lo rows get B_hi, hi rows 0
                      put(lo_row + k, hb);
                      continue;
                    }
                    put(hi_row + k, hb);
                    put(lo_row + k, lb);
                  }
          }
        }
      }
    }
}

// slot assignment and per-class entry lists for one table
void append_table(const HostTable& t, int P, int PP, int parity, std::vector<float>& coef,
                  std::vector<const double*>& slot_src, std::vector<std::vector<int4>>& cls_lists) {
  const int64_t K = (int64_t)t.active.size();
  for (int64_t i = 0; i < K; ++i) {
    if (!t.active[i]) continue;
    const int dx = (int)t.offsets[3 * i], dy = (int)t.offsets[3 * i + 1],
              dz = (int)t.offsets[3 * i + 2];
    const int slot = (int)(coef.size() / ((size_t)PP * PP));
    coef.resize(coef.size() + (size_t)PP * PP, 0.f);
    float* B = coef.data() + (size_t)slot * PP * PP;
    const double* A = t.coeffs.data() + (size_t)i * P * P;  // [k][n]
    for (int k = 0; k < P; ++k)
      for (int n = 0; n < P; ++n) B[(size_t)n * PP + k] = (float)A[(size_t)k * P + n];
    slot_src.push_back(A);
    const int ncls = (int)cls_lists.size();
    for (int c = 0; c < ncls; ++c) {
      if (parity) {
        const int par[3] = {(c >> 2) & 1, (c >> 1) & 1, c & 1};
        const int d[3] = {dx, dy, dz};
        bool ok = true;
        for (int a = 0; a < 3; ++a) {
          if (d[a] == -3 && par[a] != 1) ok = false;
          if (d[a] == 3 && par[a] != 0) ok = false;
        }
        if (!ok) continue;
      }
      cls_lists[c].push_back(make_int4(dx, dy, dz, slot));
    }
  }
}

void finish_plan(Plan& p, std::vector<std::vector<int4>>& lists) {
  p.ncls = (int)lists.size();
  p.cls_start.assign(1, 0);
  p.entries.clear();
  p.max_list = 0;
  for (auto& l : lists) {
    p.entries.insert(p.entries.end(), l.begin(), l.end());
    p.cls_start.push_back((int)p.entries.size());
    p.max_list = std::max(p.max_list, (int)l.size());
  }
  p.tc = p.ncls == 8;
}

// tensor-core M2L for a level: parity stencil and at least a 16^3 class lattice
bool use_tc(const Plan& p, int level) {
  return p.tc && p.d_tcb && p.max_list > 0 && (1 << (level + 1)) / 2 >= 16;
}

size_t tc_ws_bytes(const Plan& p, int rho, int level, int C) {
  return fc2t2::tc_workspace_bytes(rho, level, C);
}

int plan_for(const fc2t2_engine* e, int level, int table, const Plan** out) {
  if (!e || !e->uploaded) return fail(FC2T2_ESTAGE, "engine tables not uploaded");
  auto it = e->plans.find(level);
  if (it == e->plans.end()) return fail(FC2T2_ESTAGE, "no M2L table for this level");
  auto jt = it->second.find(table);
  if (jt == it->second.end()) return fail(FC2T2_ESTAGE, "table kind not available at this level");
  *out = &jt->second;
  return FC2T2_OK;
}

fc2t2::TCPlan tc_of(const fc2t2_engine* e, const Plan& p, int level) {
  fc2t2::TCPlan t;
  t.level = level;
  t.btab = p.d_tcb;
  t.rk = p.d_rk;
  t.s_inv = p.d_sinv;
  static const char* names[] = {"m2l_tc_L0", "m2l_tc_L1", "m2l_tc_L2", "m2l_tc_L3", "m2l_tc_L4",
                                "m2l_tc_L5", "m2l_tc_L6", "m2l_tc_L7", "m2l_tc_L8", "m2l_tc_L9"};
  t.level_name = names[level < 0 ? 0 : (level > 9 ? 9 : level)];
  return t;
}

fc2t2::M2LLaunch launch_of(const Plan& p, int level) {
  fc2t2::M2LLaunch l;
  l.level = level;
  l.stride = p.stride;
  l.ncls = p.ncls;
  l.entries = p.d_entries;
  l.cls_start = p.d_cls_start;
  l.max_list = p.max_list;
  static const char* names[] = {"m2l_L0", "m2l_L1", "m2l_L2", "m2l_L3", "m2l_L4",
                                "m2l_L5", "m2l_L6", "m2l_L7", "m2l_L8", "m2l_L9"};
  l.level_name = names[level < 0 ? 0 : (level > 9 ? 9 : level)];
  return l;
}

size_t grid_floats(int level, int C, int PP) {
  const size_t res = (size_t)1 << (level + 1);
  return res * res * res * (size_t)C * PP;
}

}  // namespace

extern "C" {

int fc2t2_version(void) { return 1; }

int64_t fc2t2_launch_count(void) { return fc2t2::g_launches.load(); }

int fc2t2_profile_enable(int on) {
  fc2t2::g_prof = on != 0;
  fc2t2::g_recs.clear();
  fc2t2::g_pool_used = 0;
  fc2t2::g_pending = nullptr;
  return FC2T2_OK;
}

int fc2t2_profile_read(int max_entries, char* names, double* ms, int64_t* counts) {
  std::vector<std::string> keys;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& r : fc2t2::g_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return fail(FC2T2_ECUDA, "profile sync");
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t k = 0;
    while (k < keys.size() && keys[k] != r.name) ++k;
    if (k == keys.size()) {
      keys.push_back(r.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[k] += t;
    cnt[k] += 1;
  }
  const int n = (int)std::min<size_t>(keys.size(), (size_t)max_entries);
  for (int k = 0; k < n; ++k) {
    std::snprintf(names + 32 * k, 32, "%s", keys[k].c_str());
    ms[k] = tot[k];
    counts[k] = cnt[k];
  }
  return n;
}

int fc2t2_profile_timeline(int max_entries, char* names, double* begin_ms, double* end_ms) {
  const int n = (int)std::min<size_t>(fc2t2::g_recs.size(), (size_t)max_entries);
  if (n == 0) return 0;
  const cudaEvent_t t0 = fc2t2::g_recs[0].a;
  for (int k = 0; k < n; ++k) {
    const auto& r = fc2t2::g_recs[k];
    if (cudaEventSynchronize(r.b) != cudaSuccess) return fail(FC2T2_ECUDA, "profile sync");
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, t0, r.a);
    cudaEventElapsedTime(&b, t0, r.b);
    std::snprintf(names + 32 * k, 32, "%s", r.name);
    begin_ms[k] = a;
    end_ms[k] = b;
  }
  return n;
}

const char* fc2t2_last_error(void) { return g_last_error.c_str(); }

int fc2t2_engine_create(int rho, int levels, fc2t2_engine** out) {
  if (!out) return fail(FC2T2_EVALUE, "null out pointer");
  if (rho < 1 || rho > 6) return fail(FC2T2_EORDER, "expansion order must be in [1, 6]");
  if (levels < kCoarsest || levels > 8) return fail(FC2T2_ESTAGE, "levels must be in [2, 8]");
  auto* e = new fc2t2_engine();
  e->rho = rho;
  e->levels = levels;
  e->P = fc2t2::index_count(rho);
  e->PP = fc2t2::pad4(e->P);
  *out = e;
  return FC2T2_OK;
}

void fc2t2_engine_destroy(fc2t2_engine* e) {
  if (!e) return;
  cudaFree(e->d_coef);
  if (e->side) cudaStreamDestroy(e->side);
  if (e->up) cudaStreamDestroy(e->up);
  if (e->fork) cudaEventDestroy(e->fork);
  if (e->join) cudaEventDestroy(e->join);
  for (cudaStream_t c : e->cs)
    if (c) cudaStreamDestroy(c);
  for (int l = 0; l < 10; ++l) {
    if (e->ev_m[l]) cudaEventDestroy(e->ev_m[l]);
    if (e->ev_c[l]) cudaEventDestroy(e->ev_c[l]);
  }
  for (auto& lv : e->plans)
    for (auto& t : lv.second) {
      cudaFree(t.second.d_entries);
      cudaFree(t.second.d_cls_start);
      cudaFree(t.second.d_tcb);
      cudaFree(t.second.d_rk);
      cudaFree(t.second.d_sinv);
    }
  delete e;
}

int fc2t2_engine_set_table(fc2t2_engine* e, int level, int nearfield, int64_t n_offsets,
                           const int64_t* offsets, const uint8_t* active,
                           const double* coeffs) {
  if (!e) return fail(FC2T2_EVALUE, "null engine");
  if (e->uploaded) return fail(FC2T2_ESTAGE, "engine already uploaded");
  if (level < kCoarsest || level > e->levels) return fail(FC2T2_ESTAGE, "table level out of range");
  if (nearfield && level != e->levels) return fail(FC2T2_ESTAGE, "near table must be finest level");
  HostTable& t = nearfield ? e->near : e->far[level];
  t.set = true;
  t.offsets.assign(offsets, offsets + 3 * n_offsets);
  t.active.assign(active, active + n_offsets);
  t.coeffs.assign(coeffs, coeffs + (size_t)n_offsets * e->P * e->P);
  return FC2T2_OK;
}

int fc2t2_engine_upload(fc2t2_engine* e, void* stream) {
  if (!e) return fail(FC2T2_EVALUE, "null engine");
  if (e->uploaded) return FC2T2_OK;
  if (!e->near.set) return fail(FC2T2_ESTAGE, "near table missing");
  for (int l = kCoarsest; l <= e->levels; ++l)
    if (!e->far.count(l) || !e->far[l].set) return fail(FC2T2_ESTAGE, "far table missing");
  std::vector<float> coef;
  std::vector<const double*> slot_src;
  const int P = e->P, PP = e->PP;
  // dense tensor-core tables only where use_tc can pick the plan (class lattice >= 16^3)
  auto tc_level = [](int l) { return (1 << (l + 1)) / 2 >= 16; };
  for (int l = kCoarsest; l <= e->levels; ++l) {
    const bool parity = l != kCoarsest;
    {
      std::vector<std::vector<int4>> lists(parity ? 8 : 1);
      append_table(e->far[l], P, PP, parity, coef, slot_src, lists);
      Plan& p = e->plans[l][FC2T2_TABLE_FAR];
      p.stride = parity ? 2 : 1;
      finish_plan(p, lists);
      if (p.tc && tc_level(l)) build_tc_table(lists, slot_src, P, PP, e->rho, l, p);
    }
    if (l == e->levels) {
      std::vector<std::vector<int4>> nl(1);
      append_table(e->near, P, PP, 0, coef, slot_src, nl);
      Plan& pn = e->plans[l][FC2T2_TABLE_NEAR];
      pn.stride = 1;
      finish_plan(pn, nl);
      // merged far + near: the near entries (same slots) appended to every class
      const Plan& pf = e->plans[l][FC2T2_TABLE_FAR];
      std::vector<std::vector<int4>> ml(pf.ncls);
      for (int c = 0; c < pf.ncls; ++c) {
        ml[c].assign(pf.entries.begin() + pf.cls_start[c], pf.entries.begin() + pf.cls_start[c + 1]);
        ml[c].insert(ml[c].end(), pn.entries.begin(), pn.entries.end());
      }
      Plan& pm = e->plans[l][FC2T2_TABLE_FARNEAR];
      pm.stride = pf.stride;
      finish_plan(pm, ml);
      if (pm.tc && tc_level(l)) build_tc_table(ml, slot_src, P, PP, e->rho, l, pm);
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t err;
  if (!coef.empty()) {
    err = cudaMalloc(&e->d_coef, coef.size() * sizeof(float));
    if (err != cudaSuccess) return cuda_status(err, "engine_upload malloc");
    err = cudaMemcpyAsync(e->d_coef, coef.data(), coef.size() * sizeof(float),
                          cudaMemcpyHostToDevice, s);
    if (err != cudaSuccess) return cuda_status(err, "engine_upload copy");
  }
  for (auto& lv : e->plans)
    for (auto& t : lv.second) {
      Plan& p = t.second;
      size_t ne = std::max<size_t>(p.entries.size(), 1);
      err = cudaMalloc(&p.d_entries, ne * sizeof(int4));
      if (err == cudaSuccess) err = cudaMalloc(&p.d_cls_start, p.cls_start.size() * sizeof(int));
      if (err == cudaSuccess && !p.entries.empty())
        err = cudaMemcpyAsync(p.d_entries, p.entries.data(), p.entries.size() * sizeof(int4),
                              cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess)
        err = cudaMemcpyAsync(p.d_cls_start, p.cls_start.data(), p.cls_start.size() * sizeof(int),
                              cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess && !p.tcb.empty()) {
        err = cudaMalloc(&p.d_tcb, p.tcb.size());
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(p.d_tcb, p.tcb.data(), p.tcb.size(), cudaMemcpyHostToDevice, s);
        if (err == cudaSuccess) err = cudaMalloc(&p.d_rk, p.rk.size() * sizeof(float));
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(p.d_rk, p.rk.data(), p.rk.size() * sizeof(float),
                                cudaMemcpyHostToDevice, s);
        if (err == cudaSuccess) err = cudaMalloc(&p.d_sinv, p.s_inv.size() * sizeof(float));
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(p.d_sinv, p.s_inv.data(), p.s_inv.size() * sizeof(float),
                                cudaMemcpyHostToDevice, s);
      }
      if (err != cudaSuccess) return cuda_status(err, "engine_upload plans");
    }
  err = cudaStreamSynchronize(s);
  if (err != cudaSuccess) return cuda_status(err, "engine_upload sync");
  for (auto& lv : e->plans)
    for (auto& t : lv.second) std::vector<uint8_t>().swap(t.second.tcb);
  err = cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming);
  if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming);
  int prio_lo = 0, prio_hi = 0;
  if (err == cudaSuccess) err = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int k = 0; k < 2 && err == cudaSuccess; ++k)
    err = cudaStreamCreateWithPriority(&e->cs[k], cudaStreamNonBlocking, prio_hi);
  if (err == cudaSuccess) err = cudaStreamCreateWithPriority(&e->up, cudaStreamNonBlocking, prio_hi);
  for (int l = 0; l < 10 && err == cudaSuccess; ++l) {
    err = cudaEventCreateWithFlags(&e->ev_m[l], cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->ev_c[l], cudaEventDisableTiming);
  }
  if (err != cudaSuccess) return cuda_status(err, "engine_upload streams");
  e->uploaded = true;
  return FC2T2_OK;
}

int64_t fc2t2_engine_list_entries(const fc2t2_engine* e, int level, int table) {
  const Plan* p;
  if (plan_for(e, level, table, &p) != FC2T2_OK) return -1;
  return (int64_t)p->entries.size();
}

int fc2t2_engine_get_list(const fc2t2_engine* e, int level, int table, int32_t* entries,
                          int32_t* cls_start) {
  const Plan* p;
  if (plan_for(e, level, table, &p) != FC2T2_OK) return -1;
  for (size_t i = 0; i < p->entries.size(); ++i) {
    entries[4 * i] = p->entries[i].x;
    entries[4 * i + 1] = p->entries[i].y;
    entries[4 * i + 2] = p->entries[i].z;
    entries[4 * i + 3] = p->entries[i].w;
  }
  for (size_t i = 0; i < p->cls_start.size(); ++i) cls_start[i] = p->cls_start[i];
  return p->ncls;
}

int fc2t2_find_box(int level, const float* d_pts, int64_t n, int32_t* d_box, int32_t* d_flag,
                   void* stream) {
  if (level < 0 || level > 9 || n < 0) return fail(FC2T2_EVALUE, "bad find_box arguments");
  return cuda_status(fc2t2::find_box(level, d_pts, n, d_box, d_flag, (cudaStream_t)stream),
                     "find_box");
}

size_t fc2t2_cell_sort_workspace_size(int level, int64_t n) {
  return fc2t2::cell_sort_workspace(level, n);
}

int fc2t2_cell_sort(int level, const float* d_pts, int64_t n, int32_t* d_order,
                    int32_t* d_cell_start, int32_t* d_flag, void* d_ws, size_t ws_bytes,
                    void* stream) {
  if (level < 0 || level > 9 || n < 0 || n > INT32_MAX)
    return fail(FC2T2_EVALUE, "bad cell_sort arguments");
  if (ws_bytes < fc2t2::cell_sort_workspace(level, n))
    return fail(FC2T2_EWORKSPACE, "cell_sort workspace too small");
  return cuda_status(fc2t2::cell_sort(level, d_pts, n, d_order, d_cell_start, d_flag, d_ws,
                                      ws_bytes, (cudaStream_t)stream),
                     "cell_sort");
}

int fc2t2_p2m(const fc2t2_engine* e, int channels, const float* d_pts, const float* d_w,
              const int32_t* d_order, const int32_t* d_cell_start, float* d_m_finest,
              void* stream) {
  if (!e || channels < 1) return fail(FC2T2_EVALUE, "bad p2m arguments");
  return cuda_status(fc2t2::p2m_sorted(e->rho, e->levels, channels, d_pts, d_w, d_order,
                                       d_cell_start, d_m_finest, (cudaStream_t)stream),
                     "p2m");
}

size_t fc2t2_p2m_points_workspace_size(const fc2t2_engine* e, int channels, int64_t n) {
  if (!e || channels < 1 || n < 0) return 0;
  if (fc2t2::p2m_brick_supported(e->levels, channels))
    return fc2t2::p2m_brick_workspace(e->levels, n, channels);
  // level >= 7: stable cell sort + gather P2M; order and cell starts live in
  // the workspace after the sort's own scratch
  const int64_t R = (int64_t)1 << (3 * (e->levels + 1));
  return fc2t2::cell_sort_workspace(e->levels, n) + 256 + 4 * (size_t)std::max<int64_t>(n, 1) +
         256 + 4 * (size_t)(R + 1) + 256;
}

int fc2t2_p2m_points_phase(const fc2t2_engine* e, int channels, const float* d_pts,
                           const float* d_w, int64_t n, float* d_m_finest, int32_t* d_flag,
                           void* d_ws, size_t ws_bytes, int phase, void* stream) {
  if (!e || channels < 1 || n < 0 || n > INT32_MAX) return fail(FC2T2_EVALUE, "bad p2m arguments");
  if (phase < 1 || phase > 3) return fail(FC2T2_EVALUE, "p2m phase must be 1, 2 or 3");
  if (ws_bytes < fc2t2_p2m_points_workspace_size(e, channels, n))
    return fail(FC2T2_EWORKSPACE, "p2m workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (fc2t2::p2m_brick_supported(e->levels, channels))
    return cuda_status(fc2t2::p2m_brick(e->rho, e->levels, channels, d_pts, d_w, n, d_m_finest,
                                        d_flag, d_ws, ws_bytes, s, phase),
                       "p2m_points");
  // level >= 7: the stable cell sort (points only) then the gather P2M
  const size_t sw = fc2t2::cell_sort_workspace(e->levels, n);
  char* p = (char*)d_ws + ((sw + 255) & ~(size_t)255);
  int32_t* order = (int32_t*)p;
  int32_t* start = (int32_t*)(p + ((4 * (size_t)std::max<int64_t>(n, 1) + 255) & ~(size_t)255));
  if (phase & 1) {
    int st = cuda_status(fc2t2::cell_sort(e->levels, d_pts, n, order, start, d_flag, d_ws, sw, s),
                         "p2m_points sort");
    if (st != FC2T2_OK) return st;
  }
  if (!(phase & 2)) return FC2T2_OK;
  return cuda_status(fc2t2::p2m_sorted(e->rho, e->levels, channels, d_pts, d_w, order, start,
                                       d_m_finest, s),
                     "p2m_points");
}

int fc2t2_p2m_points(const fc2t2_engine* e, int channels, const float* d_pts, const float* d_w,
                     int64_t n, float* d_m_finest, int32_t* d_flag, void* d_ws, size_t ws_bytes,
                     void* stream) {
  return fc2t2_p2m_points_phase(e, channels, d_pts, d_w, n, d_m_finest, d_flag, d_ws, ws_bytes, 3,
                                stream);
}

int fc2t2_m2m(const fc2t2_engine* e, int channels, int fine_level, const float* d_fine,
              float* d_coarse, void* stream) {
  if (!e || channels < 1) return fail(FC2T2_EVALUE, "bad m2m arguments");
  if (fine_level <= kCoarsest || fine_level > e->levels)
    return fail(FC2T2_ESTAGE, "already at the coarsest level");
  return cuda_status(
      fc2t2::m2m(e->rho, fine_level, channels, d_fine, d_coarse, (cudaStream_t)stream), "m2m");
}

int fc2t2_l2l(const fc2t2_engine* e, int channels, int coarse_level, const float* d_coarse,
              float* d_fine, int accumulate, void* stream) {
  if (!e || channels < 1) return fail(FC2T2_EVALUE, "bad l2l arguments");
  if (coarse_level < kCoarsest - 1 || coarse_level >= 9)
    return fail(FC2T2_ESTAGE, "bad l2l level");
  return cuda_status(fc2t2::l2l(e->rho, coarse_level, channels, d_coarse, d_fine, accumulate,
                                (cudaStream_t)stream),
                     "l2l");
}

double fc2t2_m2l_issued_flops(const fc2t2_engine* e, int channels, int level, int table) {
  const Plan* p;
  if (plan_for(e, level, table, &p) != FC2T2_OK || !use_tc(*p, level)) return 0.0;
  return fc2t2::tc_issued_flops(e->rho, level, channels);
}

size_t fc2t2_m2l_workspace_size(const fc2t2_engine* e, int channels, int level, int table) {
  const Plan* p;
  if (plan_for(e, level, table, &p) != FC2T2_OK) return 0;
  if (table == FC2T2_TABLE_FAR && level < e->levels && e->sep_far.count(level))
    return fc2t2::m2l_sep_workspace_floats(e->rho, level, channels, true) * sizeof(float);
  return use_tc(*p, level) ? tc_ws_bytes(*p, e->rho, level, channels) : 0;
}

int fc2t2_m2l(const fc2t2_engine* e, int channels, int level, int table, const float* d_m,
              float* d_l, int accumulate, void* d_ws, size_t ws_bytes, void* stream) {
  const Plan* p;
  int st = plan_for(e, level, table, &p);
  if (st != FC2T2_OK) return st;
  if (channels < 1) return fail(FC2T2_EVALUE, "channels must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  if (p->max_list == 0) {
    if (accumulate) return FC2T2_OK;
    return cuda_status(
        cudaMemsetAsync(d_l, 0, grid_floats(level, channels, e->PP) * sizeof(float), s), "m2l");
  }
  if (table == FC2T2_TABLE_FAR && level < e->levels && !accumulate && d_ws) {
    // a coarse level's far table through its separable factors
    auto sf = e->sep_far.find(level);
    if (sf != e->sep_far.end() &&
        ws_bytes >= fc2t2::m2l_sep_workspace_floats(e->rho, level, channels, true) * sizeof(float)) {
      const int R1 = e->rho + 1;
      const double* f = sf->second.data();
      return cuda_status(
          fc2t2::m2l_sep(e->rho, level, channels, f, f + R1 * R1, f + 2 * R1 * R1, d_m, d_l,
                         (float*)d_ws, 0, -1, s, fc2t2::SEP_ALL, nullptr, true),
          "m2l_sep far");
    }
  }
  const size_t need = use_tc(*p, level) ? tc_ws_bytes(*p, e->rho, level, channels) : 0;
  if (need && d_ws && ws_bytes >= need) {
    const fc2t2::TCPlan tp = tc_of(e, *p, level);
    st = cuda_status(fc2t2::tc_prepare(e->rho, channels, tp, d_m, d_ws, s), "m2l split");
    if (st != FC2T2_OK) return st;
    return cuda_status(fc2t2::m2l_tc(e->rho, channels, tp, d_ws, d_l, accumulate, s), "m2l_tc");
  }
  return cuda_status(
      fc2t2::m2l(e->rho, channels, launch_of(*p, level), e->d_coef, d_m, d_l, accumulate, s),
      "m2l");
}

namespace {
// scratch (floats) one M2L launch of plan p needs: tcgen05 hi/lo planes or
// split-K partial grids
size_t part_floats(const fc2t2_engine* e, const Plan& p, int level, int channels) {
  if (p.max_list == 0) return 0;
  if (level < e->levels && e->sep_far.count(level))
    return fc2t2::m2l_sep_workspace_floats(e->rho, level, channels, true);
  if (use_tc(p, level)) return (tc_ws_bytes(p, e->rho, level, channels) + 3) / 4;
  const int sp = fc2t2::m2l_splits(e->rho, channels, launch_of(p, level));
  return sp > 1 ? (size_t)sp * grid_floats(level, channels, e->PP) : 0;
}

}  // namespace

int fc2t2_engine_set_separable(fc2t2_engine* e, const double* pre, const double* post,
                               const double* conv) {
  if (!e) return fail(FC2T2_EVALUE, "null engine");
  if (!pre || !post || !conv) {
    e->sep = false;
    return FC2T2_OK;
  }
  const int res = 1 << (e->levels + 1);
  if (e->rho > 5 || e->levels <= kCoarsest || res % 32)
    return fail(FC2T2_EVALUE, "separable M2L needs rho <= 5 and a finest grid of >= 32 cells");
  const int R1 = e->rho + 1;
  e->sep_pre.assign(pre, pre + R1 * R1);
  e->sep_post.assign(post, post + R1 * R1);
  e->sep_conv.assign(conv, conv + 7 * R1 * R1);
  e->sep = true;
  return FC2T2_OK;
}

int fc2t2_engine_separable(const fc2t2_engine* e) { return e && e->sep ? 1 : 0; }

int fc2t2_engine_set_separable_far(fc2t2_engine* e, int level, const double* pre,
                                   const double* post, const double* conv) {
  if (!e) return fail(FC2T2_EVALUE, "null engine");
  if (!pre || !post || !conv) {
    e->sep_far.erase(level);
    return FC2T2_OK;
  }
  const int res = 1 << (level + 1);
  if (e->rho > 5 || level <= kCoarsest || level >= e->levels || res < 16)
    return fail(FC2T2_EVALUE,
                "separable far M2L needs rho <= 5 and a coarse level of >= 16 cells per axis");
  const int R1 = e->rho + 1;
  std::vector<double> f(9 * R1 * R1);
  std::copy(pre, pre + R1 * R1, f.begin());
  std::copy(post, post + R1 * R1, f.begin() + R1 * R1);
  std::copy(conv, conv + 7 * R1 * R1, f.begin() + 2 * R1 * R1);
  e->sep_far[level] = std::move(f);
  return FC2T2_OK;
}

int fc2t2_engine_set_sep_fusion(fc2t2_engine* e, int fuse_l2l) {
  if (!e) return fail(FC2T2_EVALUE, "null engine");
  e->sep_fuse_l2l = fuse_l2l != 0;
  return FC2T2_OK;
}

namespace {
struct ExpandLayout {
  size_t coarse_grids = 0, fine_part = 0, coarse_part = 0;
  size_t part_off[10] = {};   // per coarse level: its M2L scratch (levels run concurrently)
  size_t total() const { return coarse_grids + fine_part + coarse_part; }
};

ExpandLayout expand_layout(const fc2t2_engine* e, int channels) {
  ExpandLayout w;
  const int L = e->levels;
  for (int l = kCoarsest; l < L; ++l) {
    w.coarse_grids += 2 * grid_floats(l, channels, e->PP);
    w.part_off[l] = w.coarse_part;
    w.coarse_part += (part_floats(e, e->plans.at(l).at(FC2T2_TABLE_FAR), l, channels) + 63) / 64 * 64;
  }
  w.fine_part = e->sep ? fc2t2::m2l_sep_workspace_floats(e->rho, L, channels)
                       : part_floats(e, e->plans.at(L).at(FC2T2_TABLE_FARNEAR), L, channels);
  return w;
}

// one level's M2L (tcgen05 or FFMA split-K) into Lg, using scratch `part`,
// for target cells with x in [x_begin, x_end)
int level_m2l(const fc2t2_engine* e, int channels, int l, const Plan& p, const float* M, float* Lg,
              int accumulate, float* part, cudaStream_t s, int x_begin = 0, int x_end = -1) {
  int st;
  if (l < e->levels) {
    auto sf = e->sep_far.find(l);
    if (sf != e->sep_far.end() && !accumulate) {
      const int R1 = e->rho + 1;
      const double* f = sf->second.data();
      return cuda_status(fc2t2::m2l_sep(e->rho, l, channels, f, f + R1 * R1, f + 2 * R1 * R1, M, Lg,
                                        part, x_begin, x_end, s, fc2t2::SEP_ALL, nullptr, true),
                         "expand m2l_sep far");
    }
  }
  if (use_tc(p, l)) {
    const fc2t2::TCPlan tp = tc_of(e, p, l);
    st = cuda_status(fc2t2::tc_prepare(e->rho, channels, tp, M, part, s), "expand split");
    if (st != FC2T2_OK) return st;
    return cuda_status(
        fc2t2::m2l_tc(e->rho, channels, tp, part, Lg, accumulate, s, x_begin, x_end),
        "expand m2l_tc");
  }
  const fc2t2::M2LLaunch ml = launch_of(p, l);
  return cuda_status(fc2t2::m2l(e->rho, channels, ml, e->d_coef, M, Lg, accumulate, s, part,
                                fc2t2::m2l_splits(e->rho, channels, ml), x_begin, x_end),
                     "expand m2l");
}

// lowest level whose far table does any work (coarser grids are unused)
int lowest_level(const fc2t2_engine* e) {
  const int L = e->levels;
  for (int l = kCoarsest; l <= L; ++l) {
    const int table = (l == L) ? FC2T2_TABLE_FARNEAR : FC2T2_TABLE_FAR;
    if (e->plans.at(l).at(table).max_list > 0) return l;
  }
  return L;
}

// the finest x-slab [x0, x1) seen at level l: [x0, x1) >> (L - l), or the
// whole level when the slab does not map to whole cells there (or to the
// 4-cell granularity of the tcgen05 and separable kernels / the 2-cell parity
// stride)
void level_slab(const fc2t2_engine* e, int l, int x0, int x1, int* b, int* en) {
  const int L = e->levels, sh = L - l, res = 1 << (l + 1);
  int lb = x0 >> sh, le = x1 >> sh;
  bool ok = ((x0 >> sh) << sh) == x0 && ((x1 >> sh) << sh) == x1 && le > lb;
  if (ok && l > kCoarsest && l < L) {
    const Plan& p = e->plans.at(l).at(FC2T2_TABLE_FAR);
    // (the separable passes' TMA windows start 16-byte aligned: x % 4 == 0)
    if (use_tc(p, l) || e->sep_far.count(l)) ok = lb % 4 == 0 && le % 4 == 0;
    else ok = lb % 2 == 0 && le % 2 == 0;
  }
  if (!ok) {
    lb = 0;
    le = res;
  }
  *b = lb;
  *en = le;
}

struct Grids {
  std::vector<float*> M, L, part;
  float* fine_part = nullptr;
};

Grids carve_grids(const fc2t2_engine* e, int channels, const float* d_m, float* d_l, void* d_ws) {
  const int L = e->levels;
  const ExpandLayout lay = expand_layout(e, channels);
  Grids g;
  g.M.assign(L + 1, nullptr);
  g.L.assign(L + 1, nullptr);
  float* w = (float*)d_ws;
  for (int l = kCoarsest; l < L; ++l) {
    g.M[l] = w;
    w += grid_floats(l, channels, e->PP);
    g.L[l] = w;
    w += grid_floats(l, channels, e->PP);
  }
  g.M[L] = const_cast<float*>(d_m);
  g.L[L] = d_l;
  g.fine_part = w;
  g.part.assign(L + 1, nullptr);
  for (int l = kCoarsest; l < L; ++l) g.part[l] = w + lay.fine_part + lay.part_off[l];
  return g;
}

enum Phase { PH_ALL = 0, PH_UP = 1, PH_DOWN = 2 };

}  // namespace

size_t fc2t2_expand_workspace_size(const fc2t2_engine* e, int channels) {
  if (!e || !e->uploaded || channels < 1) return 0;
  return expand_layout(e, channels).total() * sizeof(float) + 256;
}

namespace {
// The cascade (Engine.expand_from_moments, ref expansion.py:268-281) for the
// finest targets with x in [x0, x1):
//   UP    M2M chain, each coarse level only on the slab's cells (the caller
//         all-gathers the coarse M grids afterwards, fc2t2_expand_grid_offset)
//   DOWN  coarse M2L + L2L on the slab at every level, finest M2L on the slab
//         (needs the finest M on [x0 - 3, x1 + 3)), final L2L
//   ALL   full M2M chain, then DOWN (the finest M is complete on entry)
// L_finest = M2L_finest(M_finest) + L2L(L_{finest-1}).  The coarse chain and
// the finest M2L are independent, so the finest M2L runs on the engine's side
// stream (fork/join events) and the coarse kernels fill the SMs its last wave
// leaves idle.  The summation order is fixed (M2L written first, L2L
// accumulated after the join), so results do not depend on the overlap.
int expand_phase(const fc2t2_engine* e, int channels, const float* d_m_finest, float* d_l_finest,
                 int x0, int x1, void* d_ws, size_t ws_bytes, cudaStream_t s, Phase ph) {
  if (!e || !e->uploaded) return fail(FC2T2_ESTAGE, "engine tables not uploaded");
  if (channels < 1) return fail(FC2T2_EVALUE, "channels must be >= 1");
  const int res_f = 1 << (e->levels + 1);
  if (x1 < 0) x1 = res_f;
  if (x0 < 0 || x1 > res_f || x0 > x1 || x0 % 4 || x1 % 4)
    return fail(FC2T2_EVALUE, "slab bounds must be multiples of 4 inside [0, res]");
  if (ws_bytes < fc2t2_expand_workspace_size(e, channels))
    return fail(FC2T2_EWORKSPACE, "expand workspace too small");
  const int L = e->levels;
  Grids G = carve_grids(e, channels, d_m_finest, d_l_finest, d_ws);
  const int lowest = lowest_level(e);
  const Plan& pL = e->plans.at(L).at(FC2T2_TABLE_FARNEAR);
  const bool fine = pL.max_list > 0, coarse = lowest < L;
  int st;
  if (ph == PH_UP) {
    for (int l = L; l > lowest; --l) {
      int cb, ce;
      level_slab(e, l - 1, x0, x1, &cb, &ce);
      st = cuda_status(fc2t2::m2m(e->rho, l, channels, G.M[l], G.M[l - 1], s, cb, ce),
                       "expand m2m");
      if (st != FC2T2_OK) return st;
    }
    return FC2T2_OK;
  }
  // FC2T2_SERIAL_CASCADE=1 keeps everything on the caller's stream (clean
  // per-kernel event timings for profiling)
  static const bool serial = [] {
    const char* v = std::getenv("FC2T2_SERIAL_CASCADE");
    return v && v[0] == '1';
  }();
  const bool overlap = fine && coarse && e->side && !serial;
  if (overlap) {
    st = cuda_status(cudaEventRecord(e->fork, s), "expand fork");
    if (st == FC2T2_OK) st = cuda_status(cudaStreamWaitEvent(e->side, e->fork, 0), "expand fork");
    if (st != FC2T2_OK) return st;
  }
  // separable finest M2L with the coarse chain present: its post transform
  // runs after the join with the last L2L fused into it
  const bool sep_fused = fine && e->sep && coarse && e->sep_fuse_l2l;
  if (fine) {
    if (e->sep)
      st = cuda_status(fc2t2::m2l_sep(e->rho, L, channels, e->sep_pre.data(), e->sep_post.data(),
                                      e->sep_conv.data(), G.M[L], G.L[L], G.fine_part, x0, x1,
                                      overlap ? e->side : s,
                                      sep_fused ? fc2t2::SEP_FRONT : fc2t2::SEP_ALL),
                       "expand m2l_sep");
    else
      st = level_m2l(e, channels, L, pL, G.M[L], G.L[L], 0, G.fine_part, overlap ? e->side : s,
                     x0, x1);
    if (st != FC2T2_OK) return st;
    if (overlap) {
      st = cuda_status(cudaEventRecord(e->join, e->side), "expand join");
      if (st != FC2T2_OK) return st;
    }
  }
  if (coarse) {
    // M grids of the coarse levels: the M2M chain here (ev_m[l] marks M_l),
    // or given on entry (PH_DOWN: all-gathered by the caller)
    if (ph == PH_ALL) {
      // overlapped: on the high-priority `up` stream behind the fork (every
      // ev_c[l] the caller's stream waits for below is downstream of it)
      cudaStream_t su = overlap && e->up ? e->up : s;
      if (su != s) {
        st = cuda_status(cudaStreamWaitEvent(su, e->fork, 0), "expand fork up");
        if (st != FC2T2_OK) return st;
      }
      for (int l = L; l > lowest; --l) {
        st = cuda_status(fc2t2::m2m(e->rho, l, channels, G.M[l], G.M[l - 1], su), "expand m2m");
        if (st == FC2T2_OK) st = cuda_status(cudaEventRecord(e->ev_m[l - 1], su), "expand ev_m");
        if (st != FC2T2_OK) return st;
      }
    } else {
      st = cuda_status(cudaEventRecord(e->ev_m[lowest], s), "expand ev_m");
      if (st != FC2T2_OK) return st;
    }
    // every coarse level's M2L, L_l = M2L_l(M_l), concurrently on its own
    // stream (each with its own scratch); levels without interactions start
    // from zero
    for (int l = lowest; l < L; ++l) {
      const Plan& p = e->plans.at(l).at(FC2T2_TABLE_FAR);
      int lb, le;
      level_slab(e, l, x0, x1, &lb, &le);
      cudaStream_t cl = serial ? s : e->cs[l & 1];
      const int ml = ph == PH_ALL ? l : lowest;
      st = cuda_status(cudaStreamWaitEvent(cl, e->ev_m[ml], 0), "expand wait M");
      if (st != FC2T2_OK) return st;
      if (p.max_list > 0)
        st = level_m2l(e, channels, l, p, G.M[l], G.L[l], 0, G.part[l], cl, lb, le);
      else
        st = cuda_status(cudaMemsetAsync(G.L[l], 0, grid_floats(l, channels, e->PP) * sizeof(float),
                                         cl),
                         "expand zero");
      if (st == FC2T2_OK) st = cuda_status(cudaEventRecord(e->ev_c[l], cl), "expand ev_c");
      if (st != FC2T2_OK) return st;
    }
    // the L2L chain: L_l += L2L(L_{l-1}), coarsest first (fixed order)
    st = cuda_status(cudaStreamWaitEvent(s, e->ev_c[lowest], 0), "expand wait M2L");
    if (st != FC2T2_OK) return st;
    for (int l = lowest + 1; l < L; ++l) {
      int lb, le;
      level_slab(e, l, x0, x1, &lb, &le);
      st = cuda_status(cudaStreamWaitEvent(s, e->ev_c[l], 0), "expand wait M2L");
      if (st == FC2T2_OK)
        st = cuda_status(fc2t2::l2l(e->rho, l - 1, channels, G.L[l - 1], G.L[l], 1, s, lb, le),
                         "expand l2l");
      if (st != FC2T2_OK) return st;
    }
    if (overlap) {
      st = cuda_status(cudaStreamWaitEvent(s, e->join, 0), "expand join");
      if (st != FC2T2_OK) return st;
    }
    if (sep_fused)
      st = cuda_status(fc2t2::m2l_sep(e->rho, L, channels, e->sep_pre.data(), e->sep_post.data(),
                                      e->sep_conv.data(), G.M[L], G.L[L], G.fine_part, x0, x1, s,
                                      fc2t2::SEP_POST, G.L[L - 1]),
                       "expand m2l_sep post+l2l");
    else
      st = cuda_status(
          fc2t2::l2l(e->rho, L - 1, channels, G.L[L - 1], G.L[L], fine ? 1 : 0, s, x0, x1),
          "expand l2l");
    if (st != FC2T2_OK) return st;
  } else if (!fine) {
    const size_t plane = (size_t)res_f * res_f * channels * e->PP;
    st = cuda_status(cudaMemsetAsync(G.L[L] + (size_t)x0 * plane, 0,
                                     (size_t)(x1 - x0) * plane * sizeof(float), s),
                     "expand zero");
    if (st != FC2T2_OK) return st;
  }
  return FC2T2_OK;
}
}  // namespace

int fc2t2_expand(const fc2t2_engine* e, int channels, const float* d_m_finest,
                 float* d_l_finest, void* d_ws, size_t ws_bytes, void* stream) {
  return expand_phase(e, channels, d_m_finest, d_l_finest, 0, -1, d_ws, ws_bytes,
                      (cudaStream_t)stream, PH_ALL);
}

int fc2t2_expand_slab(const fc2t2_engine* e, int channels, const float* d_m_finest,
                      float* d_l_finest, int x_begin, int x_end, void* d_ws, size_t ws_bytes,
                      void* stream) {
  return expand_phase(e, channels, d_m_finest, d_l_finest, x_begin, x_end, d_ws, ws_bytes,
                      (cudaStream_t)stream, PH_ALL);
}

int fc2t2_expand_up(const fc2t2_engine* e, int channels, const float* d_m_finest, int x_begin,
                    int x_end, void* d_ws, size_t ws_bytes, void* stream) {
  return expand_phase(e, channels, d_m_finest, nullptr, x_begin, x_end, d_ws, ws_bytes,
                      (cudaStream_t)stream, PH_UP);
}

int fc2t2_expand_down(const fc2t2_engine* e, int channels, const float* d_m_finest,
                      float* d_l_finest, int x_begin, int x_end, void* d_ws, size_t ws_bytes,
                      void* stream) {
  return expand_phase(e, channels, d_m_finest, d_l_finest, x_begin, x_end, d_ws, ws_bytes,
                      (cudaStream_t)stream, PH_DOWN);
}

int fc2t2_expand_lowest(const fc2t2_engine* e) {
  if (!e || !e->uploaded) return -1;
  return lowest_level(e);
}

int64_t fc2t2_expand_grid_offset(const fc2t2_engine* e, int channels, int level) {
  if (!e || !e->uploaded || channels < 1 || level < kCoarsest || level >= e->levels) return -1;
  size_t off = 0;
  for (int l = kCoarsest; l < level; ++l) off += 2 * grid_floats(l, channels, e->PP);
  return (int64_t)(off * sizeof(float));
}

int fc2t2_expand_slab_split(const fc2t2_engine* e, int x_begin, int x_end) {
  if (!e || !e->uploaded) return 0;
  const int L = e->levels, res_f = 1 << (L + 1);
  if (x_end < 0) x_end = res_f;
  if (x_begin < 0 || x_end > res_f || x_begin >= x_end || x_begin % 4 || x_end % 4) return 0;
  for (int l = lowest_level(e); l < L; ++l) {
    int b, en;
    level_slab(e, l, x_begin, x_end, &b, &en);
    if (b == 0 && en == (1 << (l + 1)) && !(x_begin == 0 && x_end == res_f)) return 0;
  }
  return 1;
}

int fc2t2_weighted_grad(const float* d_grad, const float* d_w, int64_t n, int channels,
                        float* d_out, void* stream) {
  if (n < 0 || channels < 1) return fail(FC2T2_EVALUE, "bad weighted_grad arguments");
  return cuda_status(fc2t2::weighted_grad(d_grad, d_w, n, channels, d_out, (cudaStream_t)stream),
                     "weighted_grad");
}

int fc2t2_l2p(int rho, int level, int channels, const float* d_l, const float* d_q, int64_t n,
              int mode, const int32_t* d_order, const float* d_wts, float* d_value,
              float* d_grad, float* d_hess, float* d_wgrad, int32_t* d_flag, void* stream) {
  if (rho < 1 || rho > 6) return fail(FC2T2_EORDER, "expansion order must be in [1, 6]");
  if (level < 0 || level > 9 || channels < 1 || n < 0) return fail(FC2T2_EVALUE, "bad l2p arguments");
  if ((mode & FC2T2_L2P_WGRAD) && !d_wts) return fail(FC2T2_EVALUE, "WGRAD needs weights");
  return cuda_status(fc2t2::l2p(rho, level, channels, d_l, d_q, n, mode, d_order, d_wts, d_value,
                                d_grad, d_hess, d_wgrad, d_flag, (cudaStream_t)stream),
                     "l2p");
}

}  // extern "C"
