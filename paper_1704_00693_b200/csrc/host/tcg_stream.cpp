// Streaming fused-chain executor: dependency analysis, sizing and CUDA code
// generation (see tcg_stream.hpp for the design).
#include "tcg_stream.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>

namespace tcg {
namespace {

constexpr int64_t kNone = -(int64_t{1} << 60);

// One dataset version: the state of a dataset after loop `prod` wrote it
// (prod = -1: the state the chain starts from, read from HBM).
struct SVer {
  int slot = -1;
  int prod = -1;
  bool needed = false;
  int64_t need[3][2] = {{kNone, kNone}, {kNone, kNone}, {kNone, kNone}};
  bool pass_only = true;     // input read only to pass unchanged points through
  std::vector<int> pass_by;  // loops passing it through
  bool store = false;
  // schedule
  int64_t lag = 0;
  int dr = 1;        // register ring depth (ages 0 .. dr-1)
  int ds = 0;        // shared-memory ring depth (0: none)
  int64_t sbase = 0; // shared-memory ring offset (rows)
  bool tma = false;  // input rows arrive by bulk copy (TMA) into the shared ring
  bool cpa = false;  // input points arrive by per-thread cp.async into the shared ring
  bool xs = false;   // read across threads (through shared memory)
  bool own_sm = false;  // the thread's own points are read from the shared ring too (no register ring)
  bool fill = false; // asynchronous input with register reads: ring filled from shared memory at age `lead`
  int lead = 1;      // input: steps between its load and the first read
  bool async_in() const { return tma || cpa; }
};

struct SRead {
  int v = -1;
  int arg = -1;
  int64_t off[3] = {0, 0, 0};
  bool pass = false;  // pass-through of a point outside the writer's range
};

struct SLoop {
  int64_t lag = 0;
  std::vector<int> vin, vout, prev;  // per argument, -1 = none
  std::vector<SRead> reads;
  bool needed = false;
  int64_t need[3][2] = {{kNone, kNone}, {kNone, kNone}, {kNone, kNone}};
};

struct Analysis {
  int dim = 2, s = 1;
  std::vector<SVer> vers;
  std::vector<SLoop> loops;
  std::vector<DatasetId> dats;  // slot -> dataset
  std::vector<int> input_ver;   // slot -> input version
  std::vector<int> final_ver;   // slot -> last version written (-1 none)
  std::vector<Range> whull;     // slot -> hull of the loops writing it
  std::vector<Range> first_w;   // slot -> range of the first writer
  std::vector<uint8_t> all_w_in_first;
  Range T, H;
  bool any_out = false;
  int64_t E[3][2] = {};
};

Range hull_or(const Range& a, bool a_set, const Range& b) { return a_set ? a.hull(b) : b; }

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
double env_dbl(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atof(e) : dflt;
}

Analysis analyze(const LoopChain& ch, const std::vector<DatasetId>& nostore = {}) {
  Analysis A;
  A.dim = ch.dim;
  A.s = ch.dim - 1;
  const int s = A.s;
  // Touched hull T: every point any loop reads or writes.
  bool tset = false;
  for (const LoopRecord& lp : ch.loops) {
    A.T = hull_or(A.T, tset, lp.range);
    tset = true;
    for (const ArgSpec& a : lp.args)
      if (mode_reads(a.mode)) {
        const Stencil& st = ch.stencil(a.stencil);
        Point lo{0, 0, 0}, hi{0, 0, 0};
        for (int d = 0; d < ch.dim; ++d) {
          lo[d] = std::min<int64_t>(st.min_offset(d), 0);
          hi[d] = std::max<int64_t>(st.max_offset(d), 0);
        }
        A.T = A.T.hull(lp.range.dilated(lo, hi));
      }
  }
  std::map<DatasetId, int> slot_of;
  auto slot = [&](DatasetId ds) {
    auto it = slot_of.find(ds);
    if (it != slot_of.end()) return it->second;
    const int k = static_cast<int>(A.dats.size());
    slot_of[ds] = k;
    A.dats.push_back(ds);
    A.input_ver.push_back(-1);
    A.final_ver.push_back(-1);
    A.whull.push_back(Range(ch.dim));
    A.first_w.push_back(Range(ch.dim));
    A.all_w_in_first.push_back(1);
    return k;
  };
  std::vector<int> cur;
  auto version_of = [&](int k) {
    if (static_cast<size_t>(k) >= cur.size()) cur.resize(static_cast<size_t>(k) + 1, -1);
    if (cur[static_cast<size_t>(k)] >= 0) return cur[static_cast<size_t>(k)];
    if (A.input_ver[static_cast<size_t>(k)] < 0) {
      SVer v;
      v.slot = k;
      A.input_ver[static_cast<size_t>(k)] = static_cast<int>(A.vers.size());
      A.vers.push_back(v);
    }
    return A.input_ver[static_cast<size_t>(k)];
  };
  // Versions, reads and pass-through edges.
  for (size_t l = 0; l < ch.loops.size(); ++l) {
    const LoopRecord& lp = ch.loops[l];
    SLoop L;
    const size_t na = lp.args.size();
    L.vin.assign(na, -1);
    L.vout.assign(na, -1);
    L.prev.assign(na, -1);
    std::vector<int> ks(na);
    for (size_t a = 0; a < na; ++a) ks[a] = slot(lp.args[a].dataset);
    for (size_t a = 0; a < na; ++a)
      for (size_t b = a + 1; b < na; ++b)
        if (ks[a] == ks[b] && mode_writes(lp.args[a].mode) && mode_writes(lp.args[b].mode))
          throw PlanError("stream executor: loop writes one dataset through two arguments");
    for (size_t a = 0; a < na; ++a) {
      if (!mode_reads(lp.args[a].mode)) continue;
      const int v = version_of(ks[a]);
      L.vin[a] = v;
      if (A.vers[static_cast<size_t>(v)].prod < 0) A.vers[static_cast<size_t>(v)].pass_only = false;
      const Stencil& st = ch.stencil(lp.args[a].stencil);
      for (const Point& p : st.points()) {
        SRead r;
        r.v = v;
        r.arg = static_cast<int>(a);
        for (int d = 0; d < 3; ++d) r.off[d] = p[d];
        L.reads.push_back(r);
      }
    }
    const bool pass = !lp.range.contains(A.T);
    for (size_t a = 0; a < na; ++a) {
      if (!mode_writes(lp.args[a].mode)) continue;
      const int k = ks[a];
      if (pass) {
        const int pv = version_of(k);
        L.prev[a] = pv;
        SRead r;
        r.v = pv;
        r.arg = static_cast<int>(a);
        r.pass = true;
        L.reads.push_back(r);
        A.vers[static_cast<size_t>(pv)].pass_by.push_back(static_cast<int>(l));
      }
      SVer nv;
      nv.slot = k;
      nv.prod = static_cast<int>(l);
      L.vout[a] = static_cast<int>(A.vers.size());
      A.vers.push_back(nv);
      const bool first = A.final_ver[static_cast<size_t>(k)] < 0;
      A.whull[static_cast<size_t>(k)] = first ? lp.range : A.whull[static_cast<size_t>(k)].hull(lp.range);
      if (first)
        A.first_w[static_cast<size_t>(k)] = lp.range;
      else if (!A.first_w[static_cast<size_t>(k)].contains(lp.range))
        A.all_w_in_first[static_cast<size_t>(k)] = 0;
      A.final_ver[static_cast<size_t>(k)] = L.vout[a];
    }
    for (size_t a = 0; a < na; ++a)
      if (L.vout[a] >= 0) {
        if (static_cast<size_t>(ks[a]) >= cur.size()) cur.resize(static_cast<size_t>(ks[a]) + 1, -1);
        cur[static_cast<size_t>(ks[a])] = L.vout[a];
      }
    A.loops.push_back(std::move(L));
  }
  // Stored versions: the final version of every written dataset.
  for (size_t k = 0; k < A.dats.size(); ++k)
    if (A.final_ver[k] >= 0 && std::find(nostore.begin(), nostore.end(), A.dats[k]) == nostore.end())
      A.vers[static_cast<size_t>(A.final_ver[k])].store = true;
  // Backward walk: the extension each version must be correct over, beyond
  // the CTA's owned box, for the stored outputs and reductions to be exact
  // (the overlapped-tile extension of construct_rank_plan, dist.cpp:268-310).
  for (SVer& v : A.vers)
    if (v.store) {
      v.needed = true;
      for (int d = 0; d < 3; ++d) v.need[d][0] = v.need[d][1] = 0;
    }
  for (size_t li = ch.loops.size(); li-- > 0;) {
    SLoop& L = A.loops[li];
    const LoopRecord& lp = ch.loops[li];
    if (lp.reduction) {
      L.needed = true;
      for (int d = 0; d < 3; ++d) L.need[d][0] = L.need[d][1] = 0;
    }
    for (int v : L.vout)
      if (v >= 0 && A.vers[static_cast<size_t>(v)].needed) {
        L.needed = true;
        for (int d = 0; d < 3; ++d)
          for (int e = 0; e < 2; ++e) L.need[d][e] = std::max(L.need[d][e], A.vers[static_cast<size_t>(v)].need[d][e]);
      }
    if (!L.needed) continue;
    for (const SRead& r : L.reads) {
      SVer& v = A.vers[static_cast<size_t>(r.v)];
      v.needed = true;
      for (int d = 0; d < 3; ++d) {
        v.need[d][0] = std::max(v.need[d][0], L.need[d][0] - r.off[d]);
        v.need[d][1] = std::max(v.need[d][1], L.need[d][1] + r.off[d]);
      }
    }
  }
  // Extension and the owned hull H (stored write hulls + reducing ranges).
  for (int d = 0; d < 3; ++d) A.E[d][0] = A.E[d][1] = 0;
  for (const SVer& v : A.vers)
    if (v.needed)
      for (int d = 0; d < A.dim; ++d)
        for (int e = 0; e < 2; ++e) A.E[d][e] = std::max(A.E[d][e], v.need[d][e]);
  bool hset = false;
  for (size_t k = 0; k < A.dats.size(); ++k)
    if (A.final_ver[k] >= 0 && A.vers[static_cast<size_t>(A.final_ver[k])].store) {
      A.H = hull_or(A.H, hset, A.whull[k]);
      hset = true;
    }
  for (size_t li = 0; li < ch.loops.size(); ++li)
    if (ch.loops[li].reduction) {
      A.H = hull_or(A.H, hset, ch.loops[li].range);
      hset = true;
    }
  A.any_out = hset && !A.H.empty();
  return A;
}

// ---------------------------------------------------------------- schedule
// Each thread owns a bx x by block of cross-section points (by = 1 in 2D).
// A read whose target point lies in another thread's block goes through a
// shared-memory ring and must target a row produced in an earlier step (age
// >= 1), so one barrier per step orders every producer before its readers.
// 2D: a thread's points are strided by the CTA width (x = x0 + tid + j*nt),
// so every in-plane neighbour belongs to another thread; 3D: a contiguous
// bx x by block (y neighbours inside it come from registers).
struct Block {
  int bx = 1, by = 1;
  bool strided = false;
  bool own_smem = false;  // reads of shared versions at age >= 1 use the smem ring (2D)
};

struct Sched {
  std::vector<SVer> vers;
  std::vector<int64_t> lag;  // per loop
  int64_t lmax = 0;
  int reg_doubles = 0;  // register-ring doubles per point
  int smem_rows = 0;    // shared-memory ring rows (planes) over all versions
  int rx = 0, ry = 0;   // in-plane reach of shared-memory reads
  int la = 1;           // bulk-copy lookahead (steps between a row's copy and its first use)
  int unroll = 1;       // step-loop unroll: every ring depth divides it
  int nbar = 0;         // mbarrier ring (0: no bulk-copied inputs)
  int ntma = 0;         // bulk-copied input versions
  int ncpa = 0;         // cp.async input versions
};

int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

bool in_block(const Block& b, const SRead& r, int dim, int jx, int jy) {
  if (r.pass) return true;
  if (b.strided && r.off[0] != 0) return false;
  const int tx = jx + static_cast<int>(r.off[0]);
  const int ty = jy + (dim == 3 ? static_cast<int>(r.off[1]) : 0);
  return tx >= 0 && tx < b.bx && ty >= 0 && ty < b.by;
}

bool crosses(const Block& b, const SRead& r, int dim) {
  for (int jy = 0; jy < b.by; ++jy)
    for (int jx = 0; jx < b.bx; ++jx)
      if (!in_block(b, r, dim, jx, jy)) return true;
  return false;
}

// Does a read of version v at `age` go through shared memory? Cross-thread
// reads always do. Reads inside the thread's block come from its register
// ring -- except, in the strided 2D layout, those of versions that are staged
// in shared memory anyway (own_smem), which saves the ring. Asynchronously
// loaded inputs land in shared memory first; their register ring (if any
// in-block read needs one) is filled from there at age `lead`.
bool read_via_smem(const SVer& v, bool in_blk, int64_t age) {
  if (!in_blk) return true;
  if (v.async_in()) return v.xs && v.own_sm;
  return v.xs && v.own_sm && age >= 1;
}

// Input transport (TCG_STREAM_INPUT): 0 = register loads `lead` steps ahead,
// 1 = TMA row copies, 2 = per-thread cp.async; 1 and 2 land in a shared ring
// `la` steps ahead of the first read.
int input_mode(int dim) {
  if (env_int("TCG_STREAM_TMA", 0) != 0) return 1;
  return env_int(dim == 2 ? "TCG_STREAM_INPUT2" : "TCG_STREAM_INPUT3", env_int("TCG_STREAM_INPUT", 2));
}

Sched schedule(const Analysis& A, const Block& B, int la) {
  Sched S;
  S.vers = A.vers;
  const int s = A.s;
  std::vector<uint8_t> shared(S.vers.size(), 0);
  for (const SLoop& L : A.loops)
    if (L.needed)
      for (const SRead& r : L.reads)
        if (crosses(B, r, A.dim)) shared[static_cast<size_t>(r.v)] = 1;
  for (size_t vi = 0; vi < S.vers.size(); ++vi) S.vers[vi].xs = shared[vi] != 0;
  const int imode = input_mode(A.dim);
  S.lag.assign(A.loops.size(), 0);
  for (size_t li = 0; li < A.loops.size(); ++li) {
    const SLoop& L = A.loops[li];
    if (!L.needed) continue;
    int64_t lag = 0;
    for (const SRead& r : L.reads) {
      const SVer& v = S.vers[static_cast<size_t>(r.v)];
      if (v.prod >= 0) lag = std::max(lag, v.lag + r.off[s] + (crosses(B, r, A.dim) ? 1 : 0));
    }
    S.lag[li] = lag;
    for (int v : L.vout)
      if (v >= 0) S.vers[static_cast<size_t>(v)].lag = lag;
  }
  // Inputs: rows read in full arrive by bulk copy `la` steps before their
  // first use; pass-through-only inputs (a few boundary points) by
  // predicated register loads one step ahead.
  for (size_t vi = 0; vi < S.vers.size(); ++vi) {
    SVer& v = S.vers[vi];
    if (v.prod >= 0 || !v.needed) continue;
    v.tma = !v.pass_only && imode == 1;
    v.cpa = !v.pass_only && imode == 2;
    const int lead = v.async_in() ? la : env_int("TCG_STREAM_REG_LEAD", A.dim == 2 ? 2 : 1);
    v.lead = lead;
    int64_t lag = int64_t{1} << 40;
    for (size_t li = 0; li < A.loops.size(); ++li) {
      if (!A.loops[li].needed) continue;
      for (const SRead& r : A.loops[li].reads)
        if (r.v == static_cast<int>(vi)) lag = std::min(lag, S.lag[li] - r.off[s] - lead);
    }
    v.lag = lag;
  }
  int64_t lmin = int64_t{1} << 40;
  for (size_t li = 0; li < A.loops.size(); ++li)
    if (A.loops[li].needed) lmin = std::min(lmin, S.lag[li]);
  for (const SVer& v : S.vers)
    if (v.needed) lmin = std::min(lmin, v.lag);
  if (lmin == (int64_t{1} << 40)) lmin = 0;
  for (int64_t& l : S.lag) l -= lmin;
  for (SVer& v : S.vers) v.lag -= lmin;
  S.lmax = 0;
  for (size_t li = 0; li < A.loops.size(); ++li)
    if (A.loops[li].needed) S.lmax = std::max(S.lmax, S.lag[li]);
  for (const SVer& v : S.vers)
    if (v.needed) S.lmax = std::max(S.lmax, v.lag);
  // Own-point reads of versions staged in shared memory: from the shared ring
  // (own_smem: no register ring, one LDS per read) or from a register ring.
  // Shared-memory bandwidth is what bounds the generated kernels (profiles/r5:
  // 62% of the crossbar on c2), so a register budget (doubles per point,
  // TCG_STREAM_OWN_BUDGET) moves the versions with the most own-point reads
  // per ring register back into registers.
  for (SVer& v : S.vers) v.own_sm = B.own_smem;
  if (B.own_smem) {
    // Measured on c2 (profiles/r5/sweeps.md): 0.569 ms/step at 0, 0.552 at 16, 0.518 at 20-24 (164
    // registers, still 3 CTAs/SM), 0.638 with every ring in registers (2 CTAs/SM).
    int budget = env_int("TCG_STREAM_OWN_BUDGET", 20);
    struct Cand {
      size_t v;
      int saved, cost;
    };
    std::vector<Cand> cands;
    for (size_t vi = 0; vi < S.vers.size(); ++vi) {
      const SVer& v = S.vers[vi];
      if (!v.needed || !v.xs) continue;
      int saved = 0;
      int64_t amax = 0;
      for (size_t li = 0; li < A.loops.size(); ++li) {
        if (!A.loops[li].needed) continue;
        for (const SRead& r : A.loops[li].reads) {
          if (r.v != static_cast<int>(vi) || !in_block(B, r, A.dim, 0, 0)) continue;
          const int64_t age = S.lag[li] - r.off[s] - v.lag;
          if (v.async_in() || age >= 1) {
            ++saved;
            amax = std::max(amax, age);
          }
        }
      }
      const int cost = v.async_in() ? static_cast<int>(amax - v.lead + 1) : static_cast<int>(amax);
      if (v.async_in()) --saved;  // the ring is filled by one shared-memory read per step
      if (saved > 0 && cost > 0) cands.push_back(Cand{vi, saved, cost});
    }
    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
      return a.saved * b.cost != b.saved * a.cost ? a.saved * b.cost > b.saved * a.cost : a.v < b.v;
    });
    for (const Cand& c : cands)
      if (c.cost <= budget) {
        S.vers[c.v].own_sm = false;
        budget -= c.cost;
      }
  }
  // Ring depths per read source.
  for (SVer& v : S.vers) {
    v.dr = v.async_in() ? 0 : 1;
    v.ds = 0;
    v.fill = false;
  }
  for (size_t li = 0; li < A.loops.size(); ++li) {
    const SLoop& L = A.loops[li];
    if (!L.needed) continue;
    for (const SRead& r : L.reads) {
      SVer& v = S.vers[static_cast<size_t>(r.v)];
      const int64_t age = S.lag[li] - r.off[s] - v.lag;
      if (age < 0) throw PlanError("stream executor: internal lag error");
      for (int jy = 0; jy < B.by; ++jy)
        for (int jx = 0; jx < B.bx; ++jx) {
          const bool blk = in_block(B, r, A.dim, jx, jy);
          const bool sm = read_via_smem(v, blk, age);
          if (sm) {
            if (age < 1) throw PlanError("stream executor: internal age error");
            v.ds = std::max<int>(v.ds, static_cast<int>(age) + 1);
            if (!blk) {
              S.rx = std::max(S.rx, std::abs(static_cast<int>(r.off[0])));
              if (A.dim == 3) S.ry = std::max(S.ry, std::abs(static_cast<int>(r.off[1])));
            }
          } else if (v.async_in()) {
            // register ring over ages lead .. age, filled from shared memory
            if (age < v.lead) throw PlanError("stream executor: internal lead error");
            v.fill = true;
            v.dr = std::max<int>(v.dr, static_cast<int>(age) - v.lead + 1);
          } else {
            v.dr = std::max<int>(v.dr, static_cast<int>(age) + 1);
          }
        }
    }
  }
  // The step loop is unrolled by a common multiple U of every ring depth, so
  // every ring slot is a compile-time index in every phase: the least common
  // multiple when it is small, else depths padded to powers of two.
  S.la = la;
  S.ntma = 0;
  S.ncpa = 0;
  for (SVer& v : S.vers) {
    if (!v.needed) continue;
    // A register-loaded shared input is staged into its ring at age lead-1.
    if (v.prod < 0 && !v.async_in() && v.ds > 0) v.dr = std::max(v.dr, v.lead);
    if (v.async_in()) v.ds = std::max(v.ds, la + 1);
    if (v.tma) ++S.ntma;
    if (v.cpa) ++S.ncpa;
  }
  S.nbar = S.ntma ? la + 1 : 0;
  auto lcm = [](int64_t a, int64_t b) {
    int64_t x = a, y = b;
    while (y) {
      const int64_t t = x % y;
      x = y;
      y = t;
    }
    return a / x * b;
  };
  int64_t L = std::max(1, S.nbar);
  for (const SVer& v : S.vers)
    if (v.needed) {
      if (v.dr > 0) L = lcm(L, v.dr);
      if (v.ds > 0) L = lcm(L, v.ds);
    }
  if (L <= env_int("TCG_STREAM_LCM_UNROLL", 8)) {
    S.unroll = static_cast<int>(L);
  } else {
    S.unroll = 1;
    for (SVer& v : S.vers) {
      if (!v.needed) continue;
      v.dr = v.dr ? pow2ceil(v.dr) : 0;
      if (v.ds > 0) v.ds = pow2ceil(v.ds);
      S.unroll = std::max({S.unroll, v.dr, v.ds});
    }
    if (S.nbar) {
      S.nbar = pow2ceil(S.nbar);
      S.unroll = std::max(S.unroll, S.nbar);
    }
  }
  if (S.ntma) S.rx = std::max(S.rx, 2);  // even-rounded copy ends overrun the tile by one
  S.reg_doubles = 0;
  S.smem_rows = 0;
  int64_t off = 0;
  for (SVer& v : S.vers) {
    if (!v.needed) continue;
    S.reg_doubles += v.dr;
    S.smem_rows += v.ds;
    v.sbase = off;  // in rows; scaled by the plane size in the sizer
    off += v.ds;
  }
  return S;
}

// ---------------------------------------------------------------- shape
struct Shape {
  Block blk;
  int nt = 256, ntx = 256;
  int tx = 512, ty = 1;
  int rx = 0, ry = 0, spx = 0;
  int64_t sp = 0;
  int64_t exl = 0, eyl = 0;  // tile origin offsets (x includes the even alignment)
  int64_t wox = 0, woy = 1;
  int64_t nxt = 1, nyt = 1, ns = 1;
  int minb = 1;
  int prefetch = 0;
  int regs = 0;
  int64_t smem_bytes = 0;
  double cost = 0;   // relative time per owned point (sizer)
  double est_s = 0;  // estimated kernel seconds (sub-chain split)
};


int est_regs(const Sched& sc, int P, int nloops) { return 2 * P * sc.reg_doubles + 6 * P + 44 + nloops / 4; }

// Picks the thread-block shape and CTA grid of one kernel (or applies the
// overrides in `c`); fills `sc` with the matching schedule. Throws PlanError
// when nothing fits.
Shape size_kernel(const Analysis& A, const LoopChain& ch, const StreamDevice& dev, const StreamChoice& c, Sched& sc) {
  const int64_t hx = A.H.extent(0), hy = A.dim == 3 ? A.H.extent(1) : 1, hs = A.H.extent(A.s);
  // Candidate shapes (measured on B200, tools/sweep_list.sh): one point per
  // thread in 2D; 32-wide warps along x with 1-4 points along y in 3D.
  const std::vector<int> nts = c.nt ? std::vector<int>{c.nt}
                                    : (A.dim == 2 ? std::vector<int>{128, 192, 256, 64} : std::vector<int>{512, 256});
  const std::vector<int> bxs = c.bx ? std::vector<int>{c.bx} : std::vector<int>{1};
  const std::vector<int> bys =
      A.dim == 2 ? std::vector<int>{1} : (c.by ? std::vector<int>{c.by} : std::vector<int>{2, 1, 4});
  const std::vector<int> ntxs = A.dim == 2 ? std::vector<int>{0} : (c.ntx ? std::vector<int>{c.ntx} : std::vector<int>{32, 16});
  int nloops = 0;
  for (const SLoop& L : A.loops) nloops += L.needed ? 1 : 0;
  const double lat_k = env_dbl("TCG_STREAM_LAT", 6.0);
  // cp.async lookahead: 2 rows in 2D (c2 0.518 -> 0.513 ms/step against 3: a smaller shared ring), 3 planes in 3D.
  const int la = std::max(1, env_int("TCG_STREAM_LOOKAHEAD", input_mode(A.dim) == 2 && A.dim == 3 ? 3 : 2));
  Shape best;
  Sched best_sc;
  best.cost = 1e300;
  bool best_good = false;
  std::map<std::pair<int, int>, Sched> scache;
  for (int bx : bxs)
    for (int by : bys) {
      Block B;
      B.bx = bx;
      B.by = by;
      // 2D: one column per thread, strided by the CTA width when a thread has
      // several; with TCG_STREAM_CONTIG2 (default on) bx > 1 means bx adjacent
      // columns (16-byte shared-memory accesses, in-register x neighbours).
      B.strided = A.dim == 2 && !(bx > 1 && bx % 2 == 0 && env_int("TCG_STREAM_CONTIG2", 1) != 0);
      B.own_smem = A.dim == 2 && env_int("TCG_STREAM_OWN_SMEM", 1) != 0;
      auto it = scache.find({bx, by});
      if (it == scache.end()) it = scache.emplace(std::make_pair(bx, by), schedule(A, B, la)).first;
      const Sched& S0 = it->second;
      for (int nt : nts)
        for (int ntx0 : ntxs) {
          Shape S;
          S.blk = B;
          S.nt = nt;
          S.ntx = A.dim == 2 ? nt : ntx0;
          if (nt % S.ntx) continue;
          const int P = bx * by;
          if (P > 16) continue;
          S.tx = S.ntx * bx;
          S.ty = A.dim == 2 ? 1 : (nt / S.ntx) * by;
          const int align = ((!B.strided && bx > 1) || S0.ntma) ? 1 : 0;
          S.exl = A.E[0][0] + align;
          S.wox = S.tx - A.E[0][0] - A.E[0][1] - align;
          if (align) S.wox &= ~int64_t{1};
          S.eyl = A.dim == 3 ? A.E[1][0] : 0;
          S.woy = A.dim == 2 ? 1 : S.ty - A.E[1][0] - A.E[1][1];
          if (S.wox <= 0 || S.woy <= 0) continue;
          S.regs = est_regs(S0, P, nloops);
          if (S.regs > 255) continue;
          S.rx = (B.strided && !S0.ntma) ? S0.rx : (S0.rx + 1) & ~1;
          S.ry = S0.ry;
          S.spx = S.tx + 2 * S.rx;
          S.sp = static_cast<int64_t>(S.spx) * (S.ty + 2 * S.ry);
          S.smem_bytes = std::max<int64_t>(S0.smem_rows * S.sp, 64) * 8;
          if (S.smem_bytes > dev.smem_optin) continue;
          S.nxt = (hx + S.wox - 1) / S.wox;
          S.nyt = A.dim == 2 ? 1 : (hy + S.woy - 1) / S.woy;
          const int rpt = (S.regs + 7) / 8 * 8;
          int cps = static_cast<int>(dev.regs_per_sm / (static_cast<int64_t>(rpt) * nt));
          cps = std::min<int>(cps, static_cast<int>(228 * 1024 / (S.smem_bytes + 1024)));
          cps = std::min(cps, 2048 / nt);
          cps = std::min(cps, 32);
          if (c.minb) cps = std::min(cps, c.minb);
          if (cps < 1) continue;
          const double red = static_cast<double>(S.nxt * S.tx) * static_cast<double>(S.nyt * S.ty) /
                             (static_cast<double>(hx) * static_cast<double>(hy));
          const double warps = cps * nt / 32.0;
          const double lat = 1.0 + lat_k / (warps * std::min(P, 4));
          S.cost = red * lat;
          S.minb = cps;
          // Measured preference order (candidates are listed best-first):
          // the first shape reaching the occupancy floor wins.
          const bool good = cps * nt >= (A.dim == 2 ? 256 : 512);
          if (good && !(best.cost < 1e300 && best_good)) {
            best = S;
            best_sc = S0;
            best_good = true;
          } else if (!best_good && S.cost < best.cost) {
            best = S;
            best_sc = S0;
          }
        }
    }
  if (best.cost >= 1e300) throw PlanError("stream executor: no thread-block shape fits the chain");
  Shape S = best;
  sc = best_sc;
  const int64_t warm = sc.lmax + A.E[A.s][0] + A.E[A.s][1];
  if (c.segments > 0) {
    S.ns = c.segments;
  } else {
    const int64_t slots = static_cast<int64_t>(dev.num_sms) * S.minb;
    const int64_t tiles = S.nxt * S.nyt;
    S.ns = std::max<int64_t>(1, slots / tiles);
    // Whole waves: round the CTA count to a multiple of the resident slots.
    if (tiles * S.ns < slots) S.ns = std::max<int64_t>(1, (slots + tiles - 1) / tiles);
    const int64_t min_len = std::max<int64_t>(8, static_cast<int64_t>(env_dbl("TCG_STREAM_MIN_SEG_WARM", 1.0) * static_cast<double>(warm)));
    S.ns = std::max<int64_t>(1, std::min<int64_t>(S.ns, hs / min_len));
  }
  S.ns = std::max<int64_t>(1, std::min<int64_t>(S.ns, hs));
  S.prefetch = c.prefetch >= 0 ? c.prefetch : 0;
  // Time estimate (sub-chain split): compute at a sustained rate of
  // cell-updates per SM clock, HBM at the copy rate; whichever is larger.
  const double red_s = 1.0 + static_cast<double>(S.ns) * static_cast<double>(warm) / static_cast<double>(std::max<int64_t>(1, hs));
  const double pts = static_cast<double>(A.H.volume());
  const double red_xy = static_cast<double>(S.nxt * S.tx) * static_cast<double>(S.nyt * S.ty) /
                        (static_cast<double>(hx) * static_cast<double>(hy));
  const double cu_clk = env_dbl("TCG_STREAM_CU_PER_CLK", 1.5);
  const double t_comp = nloops * pts * red_xy * red_s / (cu_clk * dev.num_sms * 1.9e9);
  double in_b = 0, out_b = 0;
  for (const SVer& v : sc.vers)
    if (v.needed && v.prod < 0) in_b += v.pass_only ? 0.5 : 8.0;
  for (const SVer& v : sc.vers)
    if (v.store) out_b += 8.0;
  const double t_dram = (in_b * (1.0 + 0.5 * (red_xy - 1.0)) + out_b) * pts * red_s / 6.2e12;
  S.est_s = std::max(t_comp, t_dram) * S.cost / red_xy + 4e-6;
  (void)ch;
  return S;
}

// ---------------------------------------------------------------- codegen
std::string fmt_L(int64_t v) { return std::to_string(v) + "LL"; }

struct Gen {
  const LoopChain& ch;
  const Analysis& A;
  const Sched& Sc;
  const Shape& S;
  std::vector<std::array<int64_t, 4>> boxes;
  std::set<std::pair<int, int64_t>> rings;  // (version, age) smem ring pointers used
  struct GC {
    int64_t x0, y0, z0, py, pz;
    Range alloc;
  };
  std::vector<GC> gcs;
  std::vector<int> slot_gc;

  int box_id(const Range& r) {
    const int64_t big = int64_t{1} << 30;
    std::array<int64_t, 4> b{r.start(0), r.end(0), A.dim == 3 ? r.start(1) : -big, A.dim == 3 ? r.end(1) : big};
    for (size_t i = 0; i < boxes.size(); ++i)
      if (boxes[i] == b) return static_cast<int>(i);
    boxes.push_back(b);
    return static_cast<int>(boxes.size()) - 1;
  }
  int P() const { return S.blk.bx * S.blk.by; }
  int jx(int j) const { return j % S.blk.bx; }
  int jy(int j) const { return j / S.blk.bx; }
  int xstep() const { return S.blk.strided ? S.nt : 1; }
  // Offsets of point j from the thread's first point: in the tile (smem,
  // padded row pitch spx) and in a dataset (row pitch py).
  int64_t sm_off(int j) const { return static_cast<int64_t>(jx(j)) * xstep() + static_cast<int64_t>(jy(j)) * S.spx; }
  int64_t g_off(const GC& q, int j) const {
    return static_cast<int64_t>(jx(j)) * xstep() + (A.dim == 3 ? static_cast<int64_t>(jy(j)) * q.py : 0);
  }
  int64_t s_lo(const Range& r) const { return r.start(A.s); }
  int64_t s_hi(const Range& r) const { return r.end(A.s); }
  bool is_shared(int v) const { return Sc.vers[static_cast<size_t>(v)].ds > 0; }
  std::string ring(int v, int64_t age) {
    rings.insert({v, age});
    return "rs" + std::to_string(v) + "_" + std::to_string(age);
  }
  // Expression reading version r.v at r's offset for point j of loop li in
  // unroll phase u (ring slots are static: (u - age) mod depth).
  std::string read_expr(size_t li, const SRead& r, int j, int u) {
    const SVer& v = Sc.vers[static_cast<size_t>(r.v)];
    const int64_t age = Sc.lag[li] - r.off[A.s] - v.lag;
    const int ox = r.pass ? 0 : static_cast<int>(r.off[0]);
    const int oy = r.pass ? 0 : (A.dim == 3 ? static_cast<int>(r.off[1]) : 0);
    const bool blk = in_block(S.blk, r, A.dim, jx(j), jy(j));
    const bool sm = read_via_smem(v, blk, age);
    if (!sm) {
      const int tj = (jy(j) + oy) * S.blk.bx + (jx(j) + ox);
      return "V" + std::to_string(r.v) + "[" + std::to_string(reg_slot(r.v, u, age)) + "][" + std::to_string(tj) + "]";
    }
    return "smp[" + std::to_string(sm_slot_off(r.v, u, age) + sm_off(j) + ox + static_cast<int64_t>(oy) * S.spx) + "]";
  }
  int reg_slot(int v, int u, int64_t age) const {
    const int d = Sc.vers[static_cast<size_t>(v)].dr;
    return static_cast<int>(((u - age) % d + d) % d);
  }
  int64_t sm_slot_off(int v, int u, int64_t age) const {
    const SVer& sv = Sc.vers[static_cast<size_t>(v)];
    const int64_t sl = ((u - age) % sv.ds + sv.ds) % sv.ds;
    return (sv.sbase + sl) * S.sp;
  }
};

void emit_prelude(std::ostringstream& o) {
  o << R"PRE(#include "tc_bodies.h"
namespace tcgj {
template <class TR, class RD, class WR, class CT>
struct Acc {
  RD& rd_;
  WR& wr_;
  CT& ct_;
  long long px_, py_, pz_;
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const { return rd_(a, dx, dy, dz); }
  __device__ __forceinline__ void write(int a, double v) const { wr_(a, v, 0); }
  __device__ __forceinline__ void increment(int a, double v) const { wr_(a, v, 1); }
  __device__ __forceinline__ void contribute(double v) const { ct_(v); }
  __device__ __forceinline__ long long x() const { return px_; }
  __device__ __forceinline__ long long y() const { return py_; }
  __device__ __forceinline__ long long z() const { return pz_; }
  __device__ __forceinline__ int nargs() const { return TR::nargs; }
  __device__ __forceinline__ int mode(int a) const { return TR::mode(a); }
  __device__ __forceinline__ int npts(int a) const { return TR::npts(a); }
  __device__ __forceinline__ int pt(int a, int j, int d) const { return TR::pt(a, j, d); }
  __device__ __forceinline__ bool reduces() const { return TR::red; }
};
__device__ __forceinline__ double comb(int op, double a, double b) {
  return op == 0 ? a + b : (op == 1 ? (a < b ? a : b) : (a > b ? a : b));
}
__device__ __forceinline__ double ident(int op) {
  return op == 0 ? 0.0 : (op == 1 ? __longlong_as_double(0x7ff0000000000000LL) : __longlong_as_double(0xfff0000000000000LL));
}
// Bit j: point j of the thread (x = cx0 + (j % BX) * SX, y = cy0 + j / BX)
// inside [xlo, xhi) x [ylo, yhi).
template <int P, int BX, int SX>
__device__ __forceinline__ unsigned cmask(int cx0, int cy0, int xlo, int xhi, int ylo, int yhi) {
  unsigned m = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int x = cx0 + (j % BX) * SX, y = cy0 + j / BX;
    if (x >= xlo && x < xhi && y >= ylo && y < yhi) m |= 1u << j;
  }
  return m;
}
__device__ __forceinline__ void pf_l2(const double* p, long long n) {
  const unsigned long long a0 = reinterpret_cast<unsigned long long>(p) & ~15ULL;
  const unsigned long long a1 = (reinterpret_cast<unsigned long long>(p + n) + 15ULL) & ~15ULL;
  if (a1 > a0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}
__device__ __forceinline__ unsigned su32(const void* p);
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double nanv() { return __longlong_as_double(0x7ff8dead00000000LL); }
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
                   su32(m)), "r"(parity) : "memory");
}
// global -> shared bulk copy (TMA), completion in bytes on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(mbar)) : "memory");
}
}  // namespace tcgj
)PRE";
}

// CTA partial of every reduction (warp shuffle, warp partials through sm[],
// fixed order), then the last CTA to finish folds the CTA partials in CTA
// order. Expects tid, cta, sm (>= 32 doubles), NT and A in scope.
void emit_red_epilogue(std::ostringstream& o, const std::vector<std::string>& accs, const std::vector<int>& red_ops, int nt) {
  if (!accs.empty()) {
    const int nw = nt / 32;
    o << "  __syncthreads();\n";
    for (size_t r = 0; r < accs.size(); ++r) {
      const int op = red_ops[r];
      o << "  {\n    double v = " << accs[r] << ";\n";
      o << "    #pragma unroll\n    for (int q = 16; q > 0; q >>= 1) v = tcgj::comb(" << op
        << ", v, __shfl_xor_sync(0xffffffffu, v, q));\n";
      o << "    if ((tid & 31) == 0) sm[tid >> 5] = v;\n    __syncthreads();\n";
      o << "    if (tid < 32) {\n      v = tid < " << nw << " ? sm[tid] : tcgj::ident(" << op << ");\n";
      o << "      #pragma unroll\n      for (int q = 16; q > 0; q >>= 1) v = tcgj::comb(" << op
        << ", v, __shfl_xor_sync(0xffffffffu, v, q));\n";
      o << "      if (tid == 0) A.part[" << r << " * gridDim.x + cta] = v;\n    }\n    __syncthreads();\n  }\n";
    }
    o << "  __shared__ unsigned int last;\n  __threadfence();\n";
    o << "  if (tid == 0) last = atomicAdd(A.ticket, 1u) == gridDim.x - 1 ? 1u : 0u;\n  __syncthreads();\n";
    o << "  if (last) {\n    __threadfence();\n    const int n = gridDim.x;\n";
    for (size_t r = 0; r < accs.size(); ++r) {
      const int op = red_ops[r];
      o << "    {\n      const int chunk = (n + NT - 1) / NT;\n      const int a0 = tid * chunk, a1 = a0 + chunk < n ? a0 + chunk : n;\n";
      o << "      double v = tcgj::ident(" << op << ");\n";
      o << "      for (int i = a0; i < a1; ++i) v = tcgj::comb(" << op << ", v, __ldcg(A.part + " << r << " * n + i));\n";
      o << "      #pragma unroll\n      for (int q = 16; q > 0; q >>= 1) v = tcgj::comb(" << op
        << ", v, __shfl_xor_sync(0xffffffffu, v, q));\n";
      o << "      if ((tid & 31) == 0) sm[tid >> 5] = v;\n      __syncthreads();\n";
      o << "      if (tid < 32) {\n        v = tid < " << nw << " ? sm[tid] : tcgj::ident(" << op << ");\n";
      o << "        #pragma unroll\n        for (int q = 16; q > 0; q >>= 1) v = tcgj::comb(" << op
        << ", v, __shfl_xor_sync(0xffffffffu, v, q));\n";
      o << "        if (tid == 0) A.out[" << r << "] = v;\n      }\n      __syncthreads();\n    }\n";
    }
    o << "    if (tid == 0) *A.ticket = 0u;\n  }\n";
  }
}

std::string generate(const LoopChain& ch, const Analysis& A, const Sched& Sc, const Shape& S,
                     const std::vector<StreamGeom>& geoms, const Range* red_mask, const std::vector<int32_t>& param_off,
                     int nparams, StreamKernel& K) {
  Gen g{ch, A, Sc, S, {}, {}, {}, {}};
  std::ostringstream o;
  const int P = g.P();
  const int s = A.s;
  const int U = Sc.unroll;
  const int nd = static_cast<int>(A.dats.size());
  const int BX = S.blk.bx;
  const bool contig = !S.blk.strided;
  const bool vec = contig && BX % 2 == 0;  // contiguous x pairs: 16-byte accesses
  for (int k = 0; k < nd; ++k) {
    const StreamGeom& G = geoms.at(static_cast<size_t>(A.dats[static_cast<size_t>(k)]));
    int found = -1;
    for (size_t c = 0; c < g.gcs.size(); ++c) {
      const Gen::GC& q = g.gcs[c];
      if (q.x0 == G.x0 && q.y0 == G.y0 && q.z0 == G.z0 && q.py == G.py && q.pz == G.pz && q.alloc == G.alloc)
        found = static_cast<int>(c);
    }
    if (found < 0) {
      g.gcs.push_back(Gen::GC{G.x0, G.y0, G.z0, G.py, G.pz, G.alloc});
      found = static_cast<int>(g.gcs.size()) - 1;
    }
    g.slot_gc.push_back(found);
  }
  auto srow = [&](const Gen::GC& q) { return s == 1 ? q.y0 : q.z0; };
  auto spitch = [&](const Gen::GC& q) { return s == 1 ? q.py : q.pz; };
  emit_prelude(o);
  o << "struct TcgArgs { const double* src[" << nd << "]; double* dst[" << nd
    << "]; double* part; double* out; unsigned int* ticket; long long ns; double p[" << std::max(1, nparams) << "]; };\n";
  for (size_t li = 0; li < ch.loops.size(); ++li) {
    if (!A.loops[li].needed) continue;
    const LoopRecord& lp = ch.loops[li];
    o << "struct Tr" << li << " {\n  static constexpr int nargs = " << lp.args.size() << ";\n";
    o << "  static constexpr bool red = " << (lp.reduction ? "true" : "false") << ";\n";
    o << "  static __device__ __forceinline__ int mode(int a) { switch (a) {";
    for (size_t a = 0; a < lp.args.size(); ++a) o << " case " << a << ": return " << static_cast<int>(lp.args[a].mode) << ";";
    o << " default: return -1; } }\n";
    o << "  static __device__ __forceinline__ int npts(int a) { switch (a) {";
    for (size_t a = 0; a < lp.args.size(); ++a)
      o << " case " << a << ": return " << ch.stencil(lp.args[a].stencil).points().size() << ";";
    o << " default: return 0; } }\n";
    o << "  static __device__ __forceinline__ int pt(int a, int j, int d) { switch ((a * 256 + j) * 4 + d) {";
    for (size_t a = 0; a < lp.args.size(); ++a) {
      const auto& pts = ch.stencil(lp.args[a].stencil).points();
      for (size_t j = 0; j < pts.size(); ++j)
        for (int d = 0; d < 3; ++d)
          if (pts[j][static_cast<size_t>(d)] != 0)
            o << " case " << ((a * 256 + j) * 4 + static_cast<size_t>(d)) << ": return " << pts[j][static_cast<size_t>(d)]
              << ";";
    }
    o << " default: return 0; } }\n};\n";
  }
  const int64_t hx0 = A.H.start(0), hx1 = A.H.end(0);
  const int64_t hy0 = A.dim == 3 ? A.H.start(1) : 0, hy1 = A.dim == 3 ? A.H.end(1) : 1;
  const int64_t hs0 = A.H.start(s), hs1 = A.H.end(s);
  const int64_t esl = A.E[s][0], esh = A.E[s][1];
  o << "#define NT " << S.nt << "\n#define P " << P << "\n#define BX " << BX << "\n#define BY " << S.blk.by
    << "\n#define NTX " << S.ntx << "\n#define SPX " << S.spx << "\n#define SX " << g.xstep() << "\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << S.nt << ", " << S.minb
    << ") tcg_stream(const __grid_constant__ TcgArgs A) {\n";
  o << "  extern __shared__ __align__(128) double sm[];\n";
  if (Sc.nbar) o << "  __shared__ __align__(8) unsigned long long bar[" << Sc.nbar << "];\n";
  o << "  const int tid = threadIdx.x;\n  const int tx = tid % NTX, ty = tid / NTX;\n  const int cta = blockIdx.x;\n";
  o << "  const int itx = cta % " << S.nxt << ", ity = (cta / " << S.nxt << ") % " << S.nyt << ", iseg = cta / "
    << (S.nxt * S.nyt) << ";\n";
  o << "  const int ox0 = " << hx0 << " + itx * " << S.wox << ", ox1 = min(ox0 + " << S.wox << ", " << hx1 << ");\n";
  o << "  const int oy0 = " << hy0 << " + ity * " << S.woy << ", oy1 = min(oy0 + " << S.woy << ", " << hy1 << ");\n";
  // Stream segments: A.ns, chosen at launch from the kernel's occupancy.
  o << "  const int s0 = " << hs0 << " + static_cast<int>(static_cast<long long>(iseg) * " << (hs1 - hs0)
    << " / A.ns), s1 = " << hs0 << " + static_cast<int>(static_cast<long long>(iseg + 1) * " << (hs1 - hs0)
    << " / A.ns);\n";
  // Tile origin X0 (even when rows are bulk-copied or paired: 16-byte alignment).
  if ((contig && BX > 1) || Sc.ntma)
    o << "  const int X0 = (ox0 - " << (S.exl - 1) << ") & ~1;\n";
  else
    o << "  const int X0 = ox0 - " << S.exl << ";\n";
  o << "  const int cx0 = X0 + " << (contig ? "tx * BX" : "tid") << ";\n";
  o << "  const int cy0 = " << (A.dim == 3 ? "oy0 - " + std::to_string(S.eyl) + " + ty * BY" : std::string("0")) << ";\n";
  if (contig)
    o << "  double* const smp = sm + (ty * BY + " << S.ry << ") * SPX + tx * BX + " << S.rx << ";\n";
  else
    o << "  double* const smp = sm + tid + " << S.rx << ";\n";
  o << "  (void)smp; (void)cy0; (void)oy1; (void)tx; (void)ty;\n";
  o << "  const int tstart = s0 - " << esl << ", tend = s1 + " << (esh + Sc.lmax) << ";\n";
  for (size_t c = 0; c < g.gcs.size(); ++c) {
    const Gen::GC& q = g.gcs[c];
    o << "  const long long po" << c << " = static_cast<long long>(cx0 - " << q.x0 << ")";
    if (A.dim == 3) o << " + static_cast<long long>(cy0 - " << q.y0 << ") * " << fmt_L(q.py);
    o << ";\n";
  }
  std::vector<int> loaded, tma, cpa;
  for (size_t v = 0; v < Sc.vers.size(); ++v)
    if (Sc.vers[v].needed && Sc.vers[v].prod < 0)
      (Sc.vers[v].tma ? tma : (Sc.vers[v].cpa ? cpa : loaded)).push_back(static_cast<int>(v));
  // Neighbour synchronisation (TCG_STREAM_NSYNC): a warp reads only the
  // shared-memory rows of the warps within the chain's in-plane reach, so the
  // per-step CTA barrier becomes one mbarrier per warp -- each warp arrives at
  // the end of its step (its writes published, its reads done) and waits, at
  // the top of the next step, for the warps it reads from. Warps then run up
  // to a step apart instead of in lock step.
  const int nwarps = S.nt / 32;
  const bool nsync = env_int(A.dim == 2 ? "TCG_STREAM_NSYNC2" : "TCG_STREAM_NSYNC3", env_int("TCG_STREAM_NSYNC", 0)) != 0 &&
                     tma.empty() && nwarps > 1 && S.nt % 32 == 0 && !(S.blk.strided && BX > 1);
  const int rows_per = A.dim == 3 ? S.ty : 1;
  const int nrows = static_cast<int>(tma.size()) * rows_per;  // bulk copies per step
  const int nissue = std::min(nrows, S.nt);                     // threads issuing them
  std::ostringstream ptrs, adv;
  std::vector<std::string> accs;
  std::vector<int> red_ops;
  for (size_t li = 0; li < ch.loops.size(); ++li)
    if (A.loops[li].needed && ch.loops[li].reduction) {
      accs.push_back("acc" + std::to_string(accs.size()));
      red_ops.push_back(static_cast<int>(ch.loops[li].reduction->op));
    }
  K.red_op = red_ops;
  // Pointers (row of step t0, advanced by U rows per unrolled iteration).
  for (int v : loaded) {
    const SVer& sv = Sc.vers[static_cast<size_t>(v)];
    const int c = g.slot_gc[static_cast<size_t>(sv.slot)];
    const Gen::GC& q = g.gcs[static_cast<size_t>(c)];
    (void)q;
    (void)c;
  }
  for (size_t li = 0; li < ch.loops.size(); ++li) {
    const SLoop& Lp = A.loops[li];
    if (!Lp.needed) continue;
    for (size_t a = 0; a < ch.loops[li].args.size(); ++a) {
      const int v = Lp.vout[a];
      if (v < 0) continue;
      const SVer& sv = Sc.vers[static_cast<size_t>(v)];
      if (!sv.store || !K.store[static_cast<size_t>(sv.slot)]) continue;
      const int c = g.slot_gc[static_cast<size_t>(sv.slot)];
      const Gen::GC& q = g.gcs[static_cast<size_t>(c)];
      (void)q;
      (void)c;
    }
  }
  auto stage_store = [&](std::ostringstream& b, int v, int u, int64_t age, const std::string& indent) {
    const int rs = g.reg_slot(v, u, age);
    const int64_t so = g.sm_slot_off(v, u, age);
    for (int j = 0; j < P; ++j) {
      if (vec && g.jx(j) % 2 == 0) {
        b << indent << "*reinterpret_cast<double2*>(&smp[" << (so + g.sm_off(j)) << "]) = make_double2(V" << v << "[" << rs
          << "][" << j << "], V" << v << "[" << rs << "][" << (j + 1) << "]);\n";
        ++j;
      } else {
        b << indent << "smp[" << (so + g.sm_off(j)) << "] = V" << v << "[" << rs << "][" << j << "];\n";
      }
    }
  };
  // ---- one step of phase u
  auto emit_step = [&](std::ostringstream& body, int u) {
    if (!tma.empty()) {
      // Bulk copies of this step's input rows (read from `la` steps on).
      body << "    if (t + " << Sc.la << " < tend && tid < " << nissue << ") {\n";
      body << "      unsigned long long* const mb = &bar[" << (u % Sc.nbar) << "];\n      unsigned bytes = 0;\n";
      body << "      for (int i = tid; i < " << nrows << "; i += " << nissue << ") {\n";
      body << "        const int iv = i / " << rows_per << ", iy = i - iv * " << rows_per << ";\n";
      body << "        (void)iy;\n";
      for (size_t k = 0; k < tma.size(); ++k) {
        const int v = tma[k];
        const SVer& sv = Sc.vers[static_cast<size_t>(v)];
        const Gen::GC& q = g.gcs[static_cast<size_t>(g.slot_gc[static_cast<size_t>(sv.slot)])];
        const int64_t slot = (u % sv.ds);
        body << "        if (iv == " << k << ") {\n";
        body << "          const int r = t - " << sv.lag << ";\n";
        if (A.dim == 3) body << "          const int yy = oy0 - " << S.eyl << " + iy;\n";
        body << "          const int xa = max(X0, " << q.alloc.start(0) << ") & ~1, xb = (min(X0 + " << S.tx << ", "
             << q.alloc.end(0) << ") + 1) & ~1;\n";
        body << "          if (r >= " << q.alloc.start(s) << " && r < " << q.alloc.end(s);
        if (A.dim == 3) body << " && yy >= " << q.alloc.start(1) << " && yy < " << q.alloc.end(1);
        body << " && xb > xa) {\n";
        body << "            const unsigned nb = static_cast<unsigned>(xb - xa) * 8u;\n";
        body << "            tcgj::mbar_expect_tx(mb, nb);\n            bytes += nb;\n";
        body << "            tcgj::bulk_g2s(sm + " << ((sv.sbase + slot) * S.sp + S.rx) << " + "
             << (A.dim == 3 ? "(iy + " + std::to_string(S.ry) + ") * " + std::to_string(S.spx) + " + " : std::string(""))
             << "(xa - X0), A.src[" << sv.slot << "] + static_cast<long long>(r - " << srow(q) << ") * " << fmt_L(spitch(q));
        if (A.dim == 3) body << " + static_cast<long long>(yy - " << q.y0 << ") * " << fmt_L(q.py);
        body << " + (xa - " << q.x0 << "), nb, mb);\n          }\n        }\n";
      }
      body << "      }\n      (void)bytes;\n      tcgj::mbar_arrive(mb);\n    }\n";
    }
    // optional L2 prefetch of input rows `prefetch` steps ahead
    if (S.prefetch > 0 && !loaded.empty()) {
      const int rows_per = A.dim == 3 ? S.ty : 1;
      int idx = 0;
      for (int v : loaded) {
        const SVer& sv = Sc.vers[static_cast<size_t>(v)];
        const Gen::GC& q = g.gcs[static_cast<size_t>(g.slot_gc[static_cast<size_t>(sv.slot)])];
        body << "    if (tid >= " << idx * rows_per << " && tid < " << (idx + 1) * rows_per << ") {\n";
        body << "      const int r = t + " << S.prefetch << " - " << sv.lag << ";\n";
        body << "      const int yy = " << (A.dim == 3 ? "oy0 - " + std::to_string(S.eyl) : std::string("0")) << " + (tid - "
             << idx * rows_per << ");\n";
        body << "      const int xa = max(ox0 - " << S.exl << ", " << q.alloc.start(0) << "), xb = min(ox0 - " << S.exl << " + "
             << S.tx << ", " << q.alloc.end(0) << ");\n";
        body << "      if (r >= " << q.alloc.start(s) << " && r < " << q.alloc.end(s);
        if (A.dim == 3) body << " && yy >= " << q.alloc.start(1) << " && yy < " << q.alloc.end(1);
        body << " && xb > xa) tcgj::pf_l2(A.src[" << sv.slot << "] + static_cast<long long>(r - " << srow(q) << ") * "
             << fmt_L(spitch(q));
        if (A.dim == 3) body << " + static_cast<long long>(yy - " << q.y0 << ") * " << fmt_L(q.py);
        body << " + (xa - " << q.x0 << "), xb - xa);\n    }\n";
        ++idx;
      }
    }
    // cp.async: every thread copies its points of the input row t - lag into
    // the shared ring (read from `la` steps on); one group per step.
    for (int v : cpa) {
      const SVer& sv = Sc.vers[static_cast<size_t>(v)];
      const int c = g.slot_gc[static_cast<size_t>(sv.slot)];
      const Gen::GC& q = g.gcs[static_cast<size_t>(c)];
      const int am = g.box_id(q.alloc);
      const int64_t so = g.sm_slot_off(v, u, 0);
      const int64_t ro = spitch(q) * u;
      body << "    { // cp.async version " << v << " (slot " << sv.slot << ")\n";
      body << "      const int r = t - " << sv.lag << ";\n";
      body << "      const double* __restrict__ lp" << v << " = A.src[" << sv.slot << "] + (rb" << c << " - "
           << fmt_L(spitch(q) * sv.lag) << ");\n";
      body << "      if (t + " << Sc.la << " < tend && r >= " << q.alloc.start(s) << " && r < " << q.alloc.end(s) << ") {\n";
      for (int j = 0; j < P; ++j) {
        const int64_t off = ro + g.g_off(q, j);
        if (vec && g.jx(j) % 2 == 0) {
          body << "        if (((m" << am << " >> " << j << ") & 3u) == 3u) tcgj::cp_async16(&smp[" << (so + g.sm_off(j)) << "], lp"
               << v << " + " << off << ");\n";
          body << "        else { if ((m" << am << " >> " << j << ") & 1u) tcgj::cp_async8(&smp[" << (so + g.sm_off(j)) << "], lp" << v
               << " + " << off << "); if ((m" << am << " >> " << (j + 1) << ") & 1u) tcgj::cp_async8(&smp["
               << (so + g.sm_off(j + 1)) << "], lp" << v << " + " << (off + 1) << "); }\n";
          ++j;
        } else {
          body << "        if ((m" << am << " >> " << j << ") & 1u) tcgj::cp_async8(&smp[" << (so + g.sm_off(j)) << "], lp" << v
               << " + " << off << ");\n";
        }
      }
      body << "      }\n    }\n";
    }
    if (!cpa.empty()) body << "    tcgj::cp_async_commit();\n";
    // loads: the input row t - lag lands in register age 0
    for (int v : loaded) {
      const SVer& sv = Sc.vers[static_cast<size_t>(v)];
      const int c = g.slot_gc[static_cast<size_t>(sv.slot)];
      const Gen::GC& q = g.gcs[static_cast<size_t>(c)];
      const int am = g.box_id(q.alloc);
      const int rs = g.reg_slot(v, u, 0);
      const int64_t ro = spitch(q) * u;
      body << "    { // load version " << v << " (slot " << sv.slot << ")\n";
      body << "      const int r = t - " << sv.lag << ";\n";
      body << "      const double* __restrict__ lp" << v << " = A.src[" << sv.slot << "] + (rb" << c << " - "
           << fmt_L(spitch(q) * sv.lag) << ");\n";
      body << "      if (r >= " << q.alloc.start(s) << " && r < " << q.alloc.end(s) << ") {\n";
      body << "        unsigned lm = m" << am << ";\n";
      if (sv.pass_only && !sv.pass_by.empty()) {
        body << "        unsigned inall = 0xffffffffu;\n";
        for (int li : sv.pass_by) {
          if (!A.loops[static_cast<size_t>(li)].needed) continue;
          const LoopRecord& lp = ch.loops[static_cast<size_t>(li)];
          const int rb = g.box_id(lp.range);
          body << "        if (!(r >= " << g.s_lo(lp.range) << " && r < " << g.s_hi(lp.range) << ")) inall = 0; else inall &= m"
               << rb << ";\n";
        }
        body << "        lm &= ~inall;\n";
      }
      for (int j = 0; j < P; ++j) {
        const int64_t off = ro + g.g_off(q, j);
        if (vec && g.jx(j) % 2 == 0) {
          body << "        if (((lm >> " << j << ") & 3u) == 3u) { const double2 q = __ldg(reinterpret_cast<const double2*>(lp"
               << v << " + " << off << ")); V" << v << "[" << rs << "][" << j << "] = q.x; V" << v << "[" << rs << "]["
               << (j + 1) << "] = q.y; }\n";
          body << "        else { if ((lm >> " << j << ") & 1u) V" << v << "[" << rs << "][" << j << "] = __ldg(lp" << v << " + "
               << off << "); if ((lm >> " << (j + 1) << ") & 1u) V" << v << "[" << rs << "][" << (j + 1) << "] = __ldg(lp"
               << v << " + " << (off + 1) << "); }\n";
          ++j;
        } else {
          body << "        if ((lm >> " << j << ") & 1u) V" << v << "[" << rs << "][" << j << "] = __ldg(lp" << v << " + "
               << off << ");\n";
        }
      }
      body << "      }\n    }\n";
    }
    // Whole-step interior path (TCG_STREAM_FAST): when every loop's row is in
    // range and every point of the thread is inside every loop's range, the
    // step is one straight-line block -- no per-loop range branches or
    // pass-through selects -- so the compiler overlaps the shared-memory
    // reads and the fp64 chains of all loops.
    // Measured on B200 (profiles/r5/sweeps.md): slower in 2D (c2 0.56 -> 0.70 ms/step: the long step
    // body doubles in size), 3-8% faster in 3D (c3 7.14 -> 6.56 ms/chain): on in 3D only.
    const bool step_fast =
        env_int(A.dim == 2 ? "TCG_STREAM_FAST2" : "TCG_STREAM_FAST3", env_int("TCG_STREAM_FAST", A.dim == 3 ? 1 : 0)) != 0;
    auto emit_loops = [&](bool all_fast) {
    size_t racc = 0;
    for (size_t li = 0; li < ch.loops.size(); ++li) {
      const SLoop& Lp = A.loops[li];
      if (!Lp.needed) continue;
      const LoopRecord& lp = ch.loops[li];
      const int rb = g.box_id(lp.range);
      body << "    { // loop " << li << ": body " << lp.kernel.fn.body << ", lag " << Sc.lag[li] << "\n";
      body << "      const int r = t - " << Sc.lag[li] << ";\n";
      body << "      const bool rin = r >= " << g.s_lo(lp.range) << " && r < " << g.s_hi(lp.range) << ";\n";
      body << "      const bool rown = r >= s0 && r < s1;\n      (void)rown;\n";
      std::string redacc;
      int redop = 0;
      if (lp.reduction) {
        redacc = accs[racc];
        redop = red_ops[racc];
        ++racc;
        body << "      const bool rred = rown";
        if (red_mask) body << " && r >= " << g.s_lo(*red_mask) << " && r < " << g.s_hi(*red_mask);
        body << ";\n";
        body << "      const unsigned mred = m_own" << (red_mask ? " & m" + std::to_string(g.box_id(*red_mask)) : "") << ";\n";
      }
      bool has_pass = false;
      for (size_t a = 0; a < lp.args.size(); ++a) has_pass = has_pass || (Lp.vout[a] >= 0 && Lp.prev[a] >= 0);
      auto emit_points = [&](bool fast) {
      for (int j = 0; j < P; ++j) {
        body << "      {\n";
        if (fast)
          body << "        const bool in = true;\n        (void)in;\n";
        else
          body << "        const bool in = rin && ((m" << rb << " >> " << j << ") & 1u);\n        (void)in;\n";
        for (size_t a = 0; a < lp.args.size(); ++a) {
          if (Lp.vout[a] < 0) continue;
          if (lp.args[a].mode == AccessMode::Write) {
            body << "        double o" << a << " = 0.0;\n";
          } else {
            SRead r;
            r.v = Lp.vin[a];
            r.arg = static_cast<int>(a);
            body << "        double o" << a << " = " << g.read_expr(li, r, j, u) << ";\n";
          }
        }
        if (lp.kernel.fn.body == 1 /* tcb::kGenSum */) {
          // gen_sum (tc_bodies.h) expanded here, same operations in the same
          // order: s = 0; s += every Read-arg stencil point in declaration
          // order; out = s * p[0] + 1/16; write / blend / increment the last
          // argument; contribute(out).
          body << "        {\n          double s_ = 0;\n";
          for (size_t a = 0; a < lp.args.size(); ++a) {
            if (lp.args[a].mode != AccessMode::Read) continue;
            for (const SRead& r : Lp.reads)
              if (!r.pass && r.arg == static_cast<int>(a)) body << "          s_ += " << g.read_expr(li, r, j, u) << ";\n";
          }
          body << "          const double out_ = s_ * A.p[" << param_off[li] << "] + 0.0625;\n";
          const size_t wi = lp.args.size() - 1;
          const AccessMode wm = lp.args[wi].mode;
          if (wm == AccessMode::Write)
            body << "          o" << wi << " = out_;\n";
          else if (wm == AccessMode::ReadWrite)
            body << "          o" << wi << " = 0.5 * o" << wi << " + 0.5 * out_;\n";
          else
            body << "          o" << wi << " = o" << wi << " + 0.25 * out_;\n";
          if (lp.reduction)
            body << "          " << redacc << " = (in && rred && ((mred >> " << j << ") & 1u)) ? tcgj::comb(" << redop << ", "
                 << redacc << ", out_) : " << redacc << ";\n";
          body << "        }\n";
        } else {
        body << "        {\n          auto rd = [&](int a_, int dx_, int dy_, int dz_) -> double {\n";
        for (size_t a = 0; a < lp.args.size(); ++a) {
          if (!mode_reads(lp.args[a].mode)) continue;
          if (Lp.vout[a] >= 0) {
            body << "            if (a_ == " << a << ") return o" << a << ";\n";
            continue;
          }
          body << "            if (a_ == " << a << ") {\n";
          for (const SRead& r : Lp.reads) {
            if (r.pass || r.arg != static_cast<int>(a)) continue;
            body << "              if (dx_ == " << r.off[0] << " && dy_ == " << r.off[1] << " && dz_ == " << r.off[2]
                 << ") return " << g.read_expr(li, r, j, u) << ";\n";
          }
          body << "            }\n";
        }
        body << "            return tcgj::nanv();\n          };\n";
        body << "          auto wr = [&](int a_, double v_, int inc_) {\n";
        for (size_t a = 0; a < lp.args.size(); ++a)
          if (Lp.vout[a] >= 0) body << "            if (a_ == " << a << ") o" << a << " = inc_ ? o" << a << " + v_ : v_;\n";
        body << "          };\n";
        if (lp.reduction)
          body << "          auto ct = [&](double v_) { " << redacc << " = (in && rred && ((mred >> " << j
               << ") & 1u)) ? tcgj::comb(" << redop << ", " << redacc << ", v_) : " << redacc << "; };\n";
        else
          body << "          auto ct = [&](double) {};\n";
        body << "          tcgj::Acc<Tr" << li << ", decltype(rd), decltype(wr), decltype(ct)> ac{rd, wr, ct, cx0 + "
             << static_cast<int64_t>(g.jx(j)) * g.xstep();
        if (A.dim == 2)
          body << ", r, 0LL};\n";
        else
          body << ", cy0 + " << g.jy(j) << ", r};\n";
        body << "          tcb::body_t<" << lp.kernel.fn.body << ">(ac, A.p + " << param_off[li] << ");\n        }\n";
        }
        for (size_t a = 0; a < lp.args.size(); ++a) {
          if (Lp.vout[a] < 0 || Lp.prev[a] < 0) continue;
          SRead r;
          r.v = Lp.prev[a];
          r.arg = static_cast<int>(a);
          r.pass = true;
          if (!fast) body << "        if (!in) o" << a << " = " << g.read_expr(li, r, j, u) << ";\n";
        }
        for (size_t a = 0; a < lp.args.size(); ++a)
          if (Lp.vout[a] >= 0 && Sc.vers[static_cast<size_t>(Lp.vout[a])].needed)
            body << "        V" << Lp.vout[a] << "[" << g.reg_slot(Lp.vout[a], u, 0) << "][" << j << "] = o" << a << ";\n";
        body << "      }\n";
      }
      };
      if (all_fast) {
        emit_points(true);
      } else if (has_pass && A.dim == 3) {
        // Interior fast path (3D; measured slower in 2D): every point of the thread inside the loop's
        // range this row -- no pass-through selects.
        body << "      if (rin && m" << rb << " == " << ((1u << P) - 1u) << "u) {\n";
        emit_points(true);
        body << "      } else {\n";
        emit_points(false);
        body << "      }\n";
      } else {
        emit_points(false);
      }
      for (size_t a = 0; a < lp.args.size(); ++a) {
        const int v = Lp.vout[a];
        if (v < 0 || !Sc.vers[static_cast<size_t>(v)].needed) continue;
        if (g.is_shared(v)) stage_store(body, v, u, 0, "      ");
        const SVer& sv = Sc.vers[static_cast<size_t>(v)];
        if (!sv.store || !K.store[static_cast<size_t>(sv.slot)]) continue;
        const int c = g.slot_gc[static_cast<size_t>(sv.slot)];
        const Gen::GC& q = g.gcs[static_cast<size_t>(c)];
        const Range& wh = A.whull[static_cast<size_t>(sv.slot)];
        const int wb = g.box_id(wh);
        const int rs = g.reg_slot(v, u, 0);
        const int64_t ro = spitch(q) * u;
        body << "      if (rown && r >= " << g.s_lo(wh) << " && r < " << g.s_hi(wh) << ") {\n";
        body << "        double* __restrict__ sp" << v << " = A.dst[" << sv.slot << "] + (rb" << c << " - "
             << fmt_L(spitch(q) * Sc.lag[li]) << ");\n";
        body << "        const unsigned sm_ = m_own & m" << wb << ";\n";
        for (int j = 0; j < P; ++j) {
          const int64_t off = ro + g.g_off(q, j);
          if (vec && g.jx(j) % 2 == 0) {
            body << "        if (((sm_ >> " << j << ") & 3u) == 3u) *reinterpret_cast<double2*>(sp" << v << " + " << off
                 << ") = make_double2(V" << v << "[" << rs << "][" << j << "], V" << v << "[" << rs << "][" << (j + 1)
                 << "]);\n";
            body << "        else { if ((sm_ >> " << j << ") & 1u) sp" << v << "[" << off << "] = V" << v << "[" << rs << "]["
                 << j << "]; if ((sm_ >> " << (j + 1) << ") & 1u) sp" << v << "[" << (off + 1) << "] = V" << v << "[" << rs
                 << "][" << (j + 1) << "]; }\n";
            ++j;
          } else {
            body << "        if ((sm_ >> " << j << ") & 1u) sp" << v << "[" << off << "] = V" << v << "[" << rs << "][" << j
                 << "];\n";
          }
        }
        body << "      }\n";
      }
      body << "    }\n";
    }
    };
    if (step_fast) {
      std::set<int> rbs;
      body << "    if (";
      bool first = true;
      for (size_t li = 0; li < ch.loops.size(); ++li) {
        if (!A.loops[li].needed) continue;
        const LoopRecord& lp = ch.loops[li];
        rbs.insert(g.box_id(lp.range));
        body << (first ? "" : " && ") << "(t - " << Sc.lag[li] << ") >= " << g.s_lo(lp.range) << " && (t - " << Sc.lag[li]
             << ") < " << g.s_hi(lp.range);
        first = false;
      }
      for (int rb : rbs) body << " && m" << rb << " == " << ((1u << P) - 1u) << "u";
      body << ") {\n";
      emit_loops(true);
      body << "    } else {\n";
      emit_loops(false);
      body << "    }\n";
    } else {
      emit_loops(false);
    }
    // inputs enter their shared ring at age la-1 (read from age la on)
    for (int v : loaded)
      if (g.is_shared(v)) stage_store(body, v, u, Sc.vers[static_cast<size_t>(v)].lead - 1, "    ");
  };
  // ---- emit: masks, rings, pointers, unrolled step loop
  std::ostringstream steps;
  for (int u = 0; u < U; ++u) {
    steps << "    { // phase " << u << "\n    const int t = t0 + " << u << ";\n    if (t < tend) {\n";
    if (!tma.empty()) {
      steps << "    if (t - " << Sc.la << " >= tstart) tcgj::mbar_wait(&bar[" << (((u - Sc.la) % Sc.nbar + Sc.nbar) % Sc.nbar)
            << "], static_cast<unsigned>(((t - " << Sc.la << " - tstart) / " << Sc.nbar << ") & 1));\n";
    }
    if (nsync) {
      // Two barriers per warp, alternating by step: a neighbour can complete
      // at most one more phase of the SAME barrier only after it has seen
      // this warp's next arrival, so the parity test cannot alias.
      steps << "    if (t > tstart) {\n      const int k_ = t - 1 - tstart;\n"
            << "      const unsigned par_ = static_cast<unsigned>((k_ >> 1) & 1);\n"
            << "      for (int w_ = nlo_; w_ <= nhi_; ++w_)\n        if (w_ != warp_) tcgj::mbar_wait(&nbar[2 * w_ + (k_ & 1)], par_);\n    }\n";
    } else {
      if (!cpa.empty()) steps << "    tcgj::cp_async_wait<" << (Sc.la - 1) << ">();\n";
      steps << "    __syncthreads();\n";
    }
    // asynchronous inputs: the row that becomes readable this step enters the register ring
    for (size_t v = 0; v < Sc.vers.size(); ++v) {
      const SVer& sv = Sc.vers[v];
      if (!sv.needed || sv.prod >= 0 || !sv.async_in() || !sv.fill || sv.dr == 0) continue;
      const int rs = g.reg_slot(static_cast<int>(v), u, sv.lead);
      const int64_t so = g.sm_slot_off(static_cast<int>(v), u, sv.lead);
      for (int j = 0; j < P; ++j) {
        if (vec && g.jx(j) % 2 == 0) {
          steps << "    { const double2 q = *reinterpret_cast<const double2*>(&smp[" << (so + g.sm_off(j)) << "]); V" << v << "["
                << rs << "][" << j << "] = q.x; V" << v << "[" << rs << "][" << (j + 1) << "] = q.y; }\n";
          ++j;
        } else {
          steps << "    V" << v << "[" << rs << "][" << j << "] = smp[" << (so + g.sm_off(j)) << "];\n";
        }
      }
    }
    emit_step(steps, u);
    if (nsync) {
      if (!cpa.empty()) steps << "    tcgj::cp_async_wait<" << (Sc.la - 1) << ">();\n";
      steps << "    __syncwarp();\n    if ((tid & 31) == 0) tcgj::mbar_arrive(&nbar[2 * warp_ + ((t - tstart) & 1)]);\n";
    }
    steps << "    }\n    }\n";
  }
  o << "  const unsigned m_own = tcgj::cmask<P, BX, SX>(cx0, cy0, ox0, ox1, oy0, oy1);\n  (void)m_own;\n";
  for (size_t b = 0; b < g.boxes.size(); ++b) {
    const auto& bb = g.boxes[b];
    o << "  const unsigned m" << b << " = tcgj::cmask<P, BX, SX>(cx0, cy0, " << bb[0] << ", " << bb[1] << ", " << bb[2]
      << ", " << bb[3] << ");\n";
  }
  for (size_t v = 0; v < Sc.vers.size(); ++v) {
    const SVer& sv = Sc.vers[v];
    if (!sv.needed || sv.dr == 0) continue;
    o << "  double V" << v << "[" << sv.dr << "][P];\n  #pragma unroll\n  for (int k = 0; k < " << sv.dr
      << "; ++k)\n    #pragma unroll\n    for (int j = 0; j < P; ++j) V" << v << "[k][j] = 0.0;\n";
  }
  for (size_t r = 0; r < accs.size(); ++r) o << "  double " << accs[r] << " = tcgj::ident(" << red_ops[r] << ");\n";
  o << ptrs.str();
  if (nsync) {
    o << "  __shared__ __align__(8) unsigned long long nbar[" << 2 * nwarps << "];\n";
    o << "  const int warp_ = tid >> 5;\n";
    if (S.blk.strided) {
      o << "  const int nlo_ = max(0, (32 * warp_ - " << S.rx << ") / 32), nhi_ = min(" << (nwarps - 1) << ", (32 * warp_ + 31 + "
        << S.rx << ") / 32);\n";
    } else {
      const int dyr = A.dim == 3 ? (S.ry + S.blk.by - 1) / S.blk.by : 0;
      o << "  const int nlo_ = max(0, ((32 * warp_) / NTX - " << dyr << ") * NTX / 32), nhi_ = min(" << (nwarps - 1)
        << ", (((32 * warp_ + 31) / NTX + " << dyr << ") * NTX + NTX - 1) / 32);\n";
    }
    o << "  if (tid == 0) {\n    for (int i = 0; i < " << 2 * nwarps << "; ++i) tcgj::mbar_init(&nbar[i], 1);\n";
    o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n  __syncthreads();\n";
  }
  if (Sc.nbar) {
    o << "  if (tid == 0) {\n    for (int i = 0; i < " << Sc.nbar << "; ++i) tcgj::mbar_init(&bar[i], " << nissue << ");\n";
    o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n  __syncthreads();\n";
  }
  o << "  for (int t0 = tstart; t0 < tend; t0 += " << U << ") {\n";
  for (size_t c = 0; c < g.gcs.size(); ++c)
    o << "    const long long rb" << c << " = static_cast<long long>(t0 - " << srow(g.gcs[c]) << ") * "
      << fmt_L(spitch(g.gcs[c])) << " + po" << c << ";\n";
  o << steps.str();
  o << adv.str();
  o << "  }\n";
  if (Sc.ncpa) o << "  tcgj::cp_async_wait<0>();\n";  // nothing may land in the reduction scratch
  emit_red_epilogue(o, accs, red_ops, S.nt);
  o << "}\n";
  return o.str();
}


// ---------------------------------------------------------------- horizontal fusion
// A run of consecutive loops none of which touches what another one writes
// (each written dataset is accessed only by its writer, at the iteration
// point) has no skew and no halo: the loops are independent and can run at
// every point back to back. The generated kernel is an untiled-style walk --
// one (x, y) column per thread, RUN rows / planes per thread, inputs read
// straight from HBM through the read-only path -- calling every body of the
// run at each point, so a field several loops read through the same stencil
// is fetched once (the compiler shares the loads across the bodies). c5's RHS
// loops are such a run: mass / momentum x3 / energy read the same nine fields
// through radius-2 stars.
size_t horizontal_run(const LoopChain& ch, size_t begin, size_t limit) {
  // written: datasets some loop of the run writes (always at the iteration
  // point); wide: datasets some loop reads through a non-identity stencil.
  // A loop joins when every dataset it shares with the run's writers is
  // touched at the iteration point only (a thread then sees its own earlier
  // write in a register), and nothing it writes was read elsewhere.
  std::set<DatasetId> written, wide;
  size_t e = begin;
  for (; e < ch.loops.size() && e < limit; ++e) {
    const LoopRecord& lp = ch.loops[e];
    if (lp.range.empty()) break;
    if (e > begin && !(lp.range == ch.loops[begin].range)) break;
    bool ok = true;
    std::set<DatasetId> w, wd;
    for (const ArgSpec& a : lp.args) {
      const bool ident = ch.stencil(a.stencil).is_identity();
      if (mode_writes(a.mode)) {
        if (!w.insert(a.dataset).second) ok = false;  // one dataset through two arguments
        if (wide.count(a.dataset)) ok = false;         // an earlier loop reads its neighbours
      }
      if (mode_reads(a.mode) && !ident) {
        if (written.count(a.dataset)) ok = false;      // neighbours another thread may have rewritten
        wd.insert(a.dataset);
      }
    }
    for (DatasetId d : wd)
      if (w.count(d)) ok = false;
    if (!ok) break;
    written.insert(w.begin(), w.end());
    wide.insert(wd.begin(), wd.end());
  }
  return e;
}

std::string generate_horizontal(const LoopChain& ch, const std::vector<StreamGeom>& geoms,
                                const std::vector<int32_t>& param_off, int nparams, StreamKernel& K, int ntx, int nty,
                                int run, const Range* red_mask) {
  std::ostringstream o;
  const int dim = ch.dim, s = dim - 1;
  const Range& R = ch.loops[0].range;
  const int nd = static_cast<int>(K.dats.size());
  std::map<DatasetId, int> slot_of;
  for (int k = 0; k < nd; ++k) slot_of[K.dats[static_cast<size_t>(k)]] = k;
  emit_prelude(o);
  o << "struct TcgArgs { const double* src[" << nd << "]; double* dst[" << nd
    << "]; double* part; double* out; unsigned int* ticket; long long ns; double p[" << std::max(1, nparams) << "]; };\n";
  for (size_t li = 0; li < ch.loops.size(); ++li) {
    const LoopRecord& lp = ch.loops[li];
    o << "struct Tr" << li << " {\n  static constexpr int nargs = " << lp.args.size() << ";\n  static constexpr bool red = "
      << (lp.reduction ? "true" : "false") << ";\n";
    o << "  static __device__ __forceinline__ int mode(int a) { switch (a) {";
    for (size_t a = 0; a < lp.args.size(); ++a) o << " case " << a << ": return " << static_cast<int>(lp.args[a].mode) << ";";
    o << " default: return -1; } }\n";
    o << "  static __device__ __forceinline__ int npts(int a) { switch (a) {";
    for (size_t a = 0; a < lp.args.size(); ++a)
      o << " case " << a << ": return " << ch.stencil(lp.args[a].stencil).points().size() << ";";
    o << " default: return 0; } }\n";
    o << "  static __device__ __forceinline__ int pt(int a, int j, int d) { switch ((a * 256 + j) * 4 + d) {";
    for (size_t a = 0; a < lp.args.size(); ++a) {
      const auto& pts = ch.stencil(lp.args[a].stencil).points();
      for (size_t j = 0; j < pts.size(); ++j)
        for (int d = 0; d < 3; ++d)
          if (pts[j][static_cast<size_t>(d)] != 0)
            o << " case " << ((a * 256 + j) * 4 + static_cast<size_t>(d)) << ": return " << pts[j][static_cast<size_t>(d)] << ";";
    }
    o << " default: return 0; } }\n};\n";
  }
  const int64_t nx = R.extent(0), ny = dim == 3 ? R.extent(1) : 1, nz = R.extent(s);
  const int64_t nxt = (nx + ntx - 1) / ntx, nyt = dim == 3 ? (ny + nty - 1) / nty : 1;
  // Reducing runs: every CTA ends with a partial + ticket, so a CTA walks
  // several RUN-plane chunks (at most ~16K CTAs); others keep one chunk.
  bool reduces = false;
  for (const LoopRecord& lp : ch.loops) reduces = reduces || lp.reduction.has_value();
  const int64_t nzc0 = (nz + run - 1) / run;
  const int64_t chunks = reduces ? std::max<int64_t>(1, (nxt * nyt * nzc0 + env_int("TCG_STREAM_HRED_CTAS", 16384) - 1) /
                                                            env_int("TCG_STREAM_HRED_CTAS", 16384))
                                 : 1;
  const int64_t nzc = (nzc0 + chunks - 1) / chunks;
  const int nt = ntx * (dim == 3 ? nty : 1);
  // y-band rasterisation of the (y, z-chunk) block index (3D), as the untiled walk does.
  const int64_t band = dim == 3 ? std::min<int64_t>(nyt, std::max<int64_t>(1, env_int("TCG_STREAM_HBAND", 16))) : 1;
  std::vector<std::string> accs;
  std::vector<int> red_ops;
  for (const LoopRecord& lp : ch.loops)
    if (lp.reduction) {
      accs.push_back("acc" + std::to_string(accs.size()));
      red_ops.push_back(static_cast<int>(lp.reduction->op));
    }
  K.red_op.assign(red_ops.begin(), red_ops.end());
  o << "#define NT " << nt << "\n";
  const int hminb = env_int("TCG_STREAM_HMINB", 0);  // register cap through the minimum-blocks launch bound (0 = none)
  o << "extern \"C\" __global__ void __launch_bounds__(" << nt;
  if (hminb > 0) o << ", " << hminb;
  o << ") tcg_stream(const __grid_constant__ TcgArgs A) {\n";
  if (!accs.empty()) o << "  __shared__ double sm[64];\n";
  for (size_t r = 0; r < accs.size(); ++r) o << "  double " << accs[r] << " = tcgj::ident(" << red_ops[r] << ");\n";
  o << "  const int tid = threadIdx.x;\n  const int tx = tid % " << ntx << ", ty = tid / " << ntx << ";\n  (void)ty;\n";
  o << "  const long long cta = blockIdx.x;\n  const int ix = static_cast<int>(cta % " << nxt << ");\n";
  o << "  const long long lin = cta / " << nxt << ";\n";
  if (dim == 3) {
    o << "  int iy, iz;\n  {\n    const long long full = " << (nyt / band) * band * nzc << "LL;\n";
    o << "    if (lin < full) { const long long b = lin / " << band * nzc << ", r = lin - b * " << band * nzc
      << "; iz = static_cast<int>(r / " << band << "); iy = static_cast<int>(b * " << band << " + (r - static_cast<long long>(iz) * "
      << band << ")); }\n";
    o << "    else { const long long w = " << (nyt % band) << ", r = lin - full; iz = static_cast<int>(r / w); iy = static_cast<int>("
      << (nyt / band) * band << " + (r - static_cast<long long>(iz) * w)); }\n  }\n";
  } else {
    o << "  const int iy = 0, iz = static_cast<int>(lin);\n  (void)iy;\n";
  }
  o << "  const int x = " << R.start(0) << " + ix * " << ntx << " + tx;\n";
  if (dim == 3) o << "  const int y = " << R.start(1) << " + iy * " << nty << " + ty;\n";
  o << "  if (x < " << R.end(0) << (dim == 3 ? " && y < " + std::to_string(R.end(1)) : std::string("")) << ") {\n";
  o << "  for (int c_ = 0; c_ < " << chunks << "; ++c_) {\n";
  o << "  const int z0 = " << R.start(s) << " + (iz * " << chunks << " + c_) * " << run << ";\n";
  std::vector<int64_t> pitch(static_cast<size_t>(nd)), ypitch(static_cast<size_t>(nd));
  for (int k = 0; k < nd; ++k) {
    const StreamGeom& G = geoms.at(static_cast<size_t>(K.dats[static_cast<size_t>(k)]));
    pitch[static_cast<size_t>(k)] = dim == 3 ? G.pz : G.py;
    ypitch[static_cast<size_t>(k)] = dim == 3 ? G.py : 0;
    o << "  const long long b" << k << " = static_cast<long long>(z0 - " << (dim == 3 ? G.z0 : G.y0) << ") * " << fmt_L(pitch[static_cast<size_t>(k)]);
    if (dim == 3) o << " + static_cast<long long>(y - " << G.y0 << ") * " << fmt_L(G.py);
    o << " + (x - " << G.x0 << ");\n";
    if (K.store[static_cast<size_t>(k)])
      o << "  double* __restrict__ const d" << k << " = A.dst[" << k << "] + b" << k << ";\n";
    else
      o << "  const double* __restrict__ const s" << k << " = A.src[" << k << "] + b" << k << ";\n";
  }
  o << "  #pragma unroll\n  for (int k = 0; k < " << run << "; ++k) {\n    const int z = z0 + k;\n    if (z < " << R.end(s) << ") {\n";
  // Written datasets: the point's current value lives in c<slot> from the
  // top of the point to its end (later loops of the run read it there);
  // loaded first unless the dataset's first access is a pure Write.
  {
    std::vector<char> have(static_cast<size_t>(nd), 0);
    for (const LoopRecord& lp : ch.loops)
      for (size_t a = 0; a < lp.args.size(); ++a) {
        const int k = slot_of.at(lp.args[a].dataset);
        if (!K.store[static_cast<size_t>(k)] || have[static_cast<size_t>(k)]) continue;
        have[static_cast<size_t>(k)] = 1;
        bool pure_write = lp.args[a].mode == AccessMode::Write;
        for (size_t b = 0; b < lp.args.size(); ++b)
          if (lp.args[b].dataset == lp.args[a].dataset && mode_reads(lp.args[b].mode)) pure_write = false;
        o << "    double c" << k << " = "
          << (pure_write ? std::string("0.0") : "d" + std::to_string(k) + "[k * " + fmt_L(pitch[static_cast<size_t>(k)]) + "]") << ";\n";
      }
  }
  size_t racc = 0;
  for (size_t li = 0; li < ch.loops.size(); ++li) {
    const LoopRecord& lp = ch.loops[li];
    o << "    { // loop " << li << ": body " << lp.kernel.fn.body << "\n";
    for (size_t a = 0; a < lp.args.size(); ++a) {
      if (!mode_writes(lp.args[a].mode)) continue;
      const int k = slot_of.at(lp.args[a].dataset);
      o << "      double o" << a << " = " << (lp.args[a].mode == AccessMode::Write ? std::string("0.0") : "c" + std::to_string(k)) << ";\n";
    }
    o << "      auto rd = [&](int a_, int dx_, int dy_, int dz_) -> double {\n";
    for (size_t a = 0; a < lp.args.size(); ++a) {
      if (!mode_reads(lp.args[a].mode)) continue;
      if (mode_writes(lp.args[a].mode)) {
        o << "        if (a_ == " << a << ") return o" << a << ";\n";
        continue;
      }
      const int k = slot_of.at(lp.args[a].dataset);
      if (K.store[static_cast<size_t>(k)]) {  // written by a loop of the run: identity reads only (horizontal_run)
        o << "        if (a_ == " << a << ") return c" << k << ";\n";
        continue;
      }
      // dim 2: (dx, dy) with dy along the walk; dim 3: dz along the walk
      if (dim == 3)
        o << "        if (a_ == " << a << ") return __ldg(s" << k << " + ((k + dz_) * " << fmt_L(pitch[static_cast<size_t>(k)]) << " + dy_ * "
          << fmt_L(ypitch[static_cast<size_t>(k)]) << " + dx_));\n";
      else
        o << "        if (a_ == " << a << ") return __ldg(s" << k << " + ((k + dy_) * " << fmt_L(pitch[static_cast<size_t>(k)]) << " + dx_));\n";
    }
    o << "        return tcgj::nanv();\n      };\n";
    o << "      auto wr = [&](int a_, double v_, int inc_) {\n";
    for (size_t a = 0; a < lp.args.size(); ++a)
      if (mode_writes(lp.args[a].mode)) o << "        if (a_ == " << a << ") o" << a << " = inc_ ? o" << a << " + v_ : v_;\n";
    o << "      };\n";
    if (lp.reduction) {
      const std::string& acc = accs[racc];
      const int op = red_ops[racc];
      ++racc;
      std::string cond = "true";
      if (red_mask) {
        cond = "x >= " + std::to_string(red_mask->start(0)) + " && x < " + std::to_string(red_mask->end(0));
        if (dim == 3) cond += " && y >= " + std::to_string(red_mask->start(1)) + " && y < " + std::to_string(red_mask->end(1));
        cond += " && z >= " + std::to_string(red_mask->start(s)) + " && z < " + std::to_string(red_mask->end(s));
      }
      o << "      auto ct = [&](double v_) { if (" << cond << ") " << acc << " = tcgj::comb(" << op << ", " << acc << ", v_); };\n";
    } else {
      o << "      auto ct = [&](double) {};\n";
    }
    o << "      tcgj::Acc<Tr" << li << ", decltype(rd), decltype(wr), decltype(ct)> ac{rd, wr, ct, x, "
      << (dim == 3 ? "y, z" : "z, 0LL") << "};\n";
    o << "      tcb::body_t<" << lp.kernel.fn.body << ">(ac, A.p + " << param_off[li] << ");\n";
    for (size_t a = 0; a < lp.args.size(); ++a) {
      if (!mode_writes(lp.args[a].mode)) continue;
      const int k = slot_of.at(lp.args[a].dataset);
      o << "      c" << k << " = o" << a << ";\n";
    }
    o << "    }\n";
  }
  for (int k = 0; k < nd; ++k)
    if (K.store[static_cast<size_t>(k)]) o << "    d" << k << "[k * " << fmt_L(pitch[static_cast<size_t>(k)]) << "] = c" << k << ";\n";
  o << "    }\n  }\n  }\n  }\n";
  emit_red_epilogue(o, accs, red_ops, nt);
  o << "}\n";
  K.nt = nt;
  K.minb = 1;
  K.smem_bytes = 0;
  K.tiles = nxt * nyt * nzc;
  K.nctas = K.tiles;
  K.forced_segments = 1;
  K.stream_extent = 1;
  K.tile[0] = ntx;
  K.tile[1] = dim == 3 ? nty : 1;
  K.owned[0] = ntx;
  K.owned[1] = dim == 3 ? nty : 1;
  K.grid[0] = static_cast<int>(nxt);
  K.grid[1] = static_cast<int>(nyt);
  K.grid[2] = static_cast<int>(nzc);
  return o.str();
}

uint64_t fnv(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

LoopChain slice_chain(const LoopChain& ch, size_t b, size_t e) {
  LoopChain s;
  s.dim = ch.dim;
  s.stencils = ch.stencils;
  s.loops.assign(ch.loops.begin() + static_cast<std::ptrdiff_t>(b), ch.loops.begin() + static_cast<std::ptrdiff_t>(e));
  return s;
}

// Is dataset ds's state after loop `end` of `ch` overwritten, before any
// read, by a later loop whose range covers `box`? Then a kernel ending at
// `end` need not store it (the later kernel of the same flush recomputes it).
bool dead_after(const LoopChain& ch, size_t end, DatasetId ds, const Range& box) {
  for (size_t l = end; l < ch.loops.size(); ++l) {
    const LoopRecord& lp = ch.loops[l];
    bool reads = false, writes_w = false;
    for (const ArgSpec& a : lp.args) {
      if (a.dataset != ds) continue;
      if (mode_reads(a.mode)) reads = true;
      if (a.mode == AccessMode::Write) writes_w = true;
    }
    if (reads) return false;
    if (writes_w) return lp.range.contains(box);
  }
  return false;
}

}  // namespace

int64_t StreamKernel::segments_for(int64_t slots) const {
  if (forced_segments > 0) return std::min<int64_t>(forced_segments, stream_extent);
  // One wave when the tiles leave room (floor: never one CTA past a wave),
  // segments long against the pipeline warm-up.
  // More tiles than resident slots: several waves. A few segments per tile
  // even out the last wave (c3, 400 tiles on 148 SMs: 7.60 ms/chain with 1
  // segment, 6.95 with 3, 6.83 with 4; profiles/r5/sweeps.md).
  int64_t ns = tiles >= slots ? (dim == 3 ? 4 : 1) : slots / tiles;
  ns = std::min<int64_t>(ns, std::max<int64_t>(1, stream_extent / min_seg));
  return std::max<int64_t>(1, ns);
}

std::string StreamKernel::cta_text(int64_t ns) const {
  std::ostringstream o;
  if (nctas == 0 && tiles <= 1 && hull.dim() == 0) return o.str();
  const int s = dim - 1;
  const int64_t nxt = grid[0], nyt = dim == 3 ? grid[1] : 1;
  int64_t idx = 0;
  for (int64_t iseg = 0; iseg < ns; ++iseg)
    for (int64_t ity = 0; ity < nyt; ++ity)
      for (int64_t itx = 0; itx < nxt; ++itx, ++idx) {
        Range own(dim);
        const int64_t ox0 = hull.start(0) + itx * owned[0];
        own.set_raw(0, ox0, std::min(ox0 + owned[0], hull.end(0)));
        if (dim == 3) {
          const int64_t oy0 = hull.start(1) + ity * owned[1];
          own.set_raw(1, oy0, std::min(oy0 + owned[1], hull.end(1)));
        }
        const int64_t ext = hull.extent(s);
        own.set_raw(s, hull.start(s) + iseg * ext / ns, hull.start(s) + (iseg + 1) * ext / ns);
        for (size_t l = 0; l < loop_range.size(); ++l) {
          Range r(dim);
          for (int d = 0; d < dim; ++d) r.set_raw(d, 0, 0);
          if (loop_live[l] && !own.empty()) {
            r = own;
            for (int d = 0; d < dim; ++d)
              r.set_raw(d, own.start(d) - loop_need[l][static_cast<size_t>(2 * d)], own.end(d) + loop_need[l][static_cast<size_t>(2 * d + 1)]);
            r = r.intersect(loop_range[l]);
          }
          o << "cta=" << idx << " loop=" << (begin + l) << " owned=" << own.to_string() << " range=" << r.to_string() << "\n";
        }
      }
  return o.str();
}

std::string StreamPlan::summary() const {
  std::ostringstream o;
  for (const StreamKernel& k : kernels) {
    o << "kernel loops=[" << k.begin << "," << k.end << ") nt=" << k.nt << " bx=" << k.bx << " by=" << k.by
      << " tile=" << k.tile[0] << "x" << k.tile[1] << " owned=" << k.owned[0] << "x" << k.owned[1] << " grid=" << k.grid[0]
      << "x" << k.grid[1] << "x" << k.grid[2] << " ctas=" << k.nctas << " minb=" << k.minb << " smem=" << k.smem_bytes
      << " lag=" << k.lag_max << " ring=" << k.ring_doubles << " smem_rows=" << k.smem_stages << " ext=";
    for (int d = 0; d < k.dim; ++d) o << (d ? "," : "") << k.ext[d][0] << "/" << k.ext[d][1];
    o << " computed=" << k.computed_points << " recorded=" << k.recorded_points << " stored=";
    for (size_t i = 0; i < k.dats.size(); ++i)
      if (k.store[i]) o << k.dats[i] << (k.pingpong[i] ? "p" : "i") << ";";
    o << "\n";
  }
  return o.str();
}

StreamPlan build_stream_plan(const LoopChain& chain, const std::vector<StreamGeom>& geoms, const StreamDevice& dev,
                             const StreamChoice& choice_in, const Range* red_mask) {
  const auto t0 = std::chrono::steady_clock::now();
  if (chain.dim < 2) throw PlanError("stream executor: 1D chains are not streamed");
  StreamChoice choice = choice_in;
  if (const char* e = std::getenv("TCG_STREAM_CFG")) {
    // nt,bx,by,ntx,segments,max_loops,minb,prefetch
    int v[8] = {0, 0, 0, 0, 0, 0, 0, -1};
    std::sscanf(e, "%d,%d,%d,%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &v[7]);
    if (v[0]) choice.nt = v[0];
    if (v[1]) choice.bx = v[1];
    if (v[2]) choice.by = v[2];
    if (v[3]) choice.ntx = v[3];
    if (v[4]) choice.segments = v[4];
    if (v[5]) choice.max_loops = v[5];
    if (v[6]) choice.minb = v[6];
    if (v[7] >= 0) choice.prefetch = v[7];
  }
  StreamPlan plan;
  const size_t L = chain.size();
  const size_t hmax = choice.max_loops > 0 ? static_cast<size_t>(choice.max_loops)
                                           : static_cast<size_t>(env_int("TCG_STREAM_MAX_LOOPS", 32));
  // Datasets whose state after loop `end` a later loop of this flush
  // overwrites before reading: kernels ending there need not store them.
  auto nostore_at = [&](size_t b, size_t e) {
    std::vector<DatasetId> ns;
    const LoopChain sub = slice_chain(chain, b, e);
    const Analysis A = analyze(sub);
    for (size_t k = 0; k < A.dats.size(); ++k)
      if (A.final_ver[k] >= 0 && dead_after(chain, e, A.dats[k], A.whull[k])) ns.push_back(A.dats[k]);
    return ns;
  };
  size_t begin = 0;
  const int horiz = env_int(chain.dim == 2 ? "TCG_STREAM_HORIZ2" : "TCG_STREAM_HORIZ3", env_int("TCG_STREAM_HORIZ", 1));
  const int hmaxl = std::max(2, env_int("TCG_STREAM_HMAXLOOPS", 12));  // loops per horizontal run
  while (begin < L) {
    // Sub-chain length (rule measured on B200): the longest
    // prefix that fits the register / shared-memory budget while the
    // overlapped tile's cross-section redundancy stays under a bound (fusing
    // more loops saves HBM traffic but widens the halo every loop
    // recomputes); in 3D at most TCG_STREAM_H3D loops.
    size_t best_end = 0;
    const size_t cap3 = chain.dim == 3 ? static_cast<size_t>(env_int("TCG_STREAM_H3D", 3)) : L;
    const size_t last = std::min({L, begin + hmax, begin + (choice.max_loops > 0 ? hmax : cap3)});
    const double rmax = env_dbl(chain.dim == 2 ? "TCG_STREAM_RMAX2" : "TCG_STREAM_RMAX3", chain.dim == 2 ? 1.15 : 1.7);
    for (size_t end = begin + 1; end <= last; ++end) {
      const LoopChain sub = slice_chain(chain, begin, end);
      const Analysis A = analyze(sub, nostore_at(begin, end));
      if (!A.any_out) {
        best_end = end;
        continue;
      }
      Sched sc;
      Shape S;
      try {
        S = size_kernel(A, sub, dev, choice, sc);
      } catch (const PlanError&) {
        break;  // longer prefixes only need more
      }
      const double hx = static_cast<double>(A.H.extent(0)), hy = A.dim == 3 ? static_cast<double>(A.H.extent(1)) : 1.0;
      const double red = static_cast<double>(S.nxt * S.tx) * static_cast<double>(S.nyt * S.ty) / (hx * hy);
      if (end > begin + 1 && red > rmax && choice.max_loops == 0) break;
      best_end = end;
    }
    if (best_end == 0) throw PlanError("stream executor: a single loop does not fit");
    // Horizontal runs (independent / own-point-dependent loops over one
    // range, fused point by point). A vertical prefix that ends inside a
    // later run of three or more loops is cut back to the run's first loop;
    // the run starting here wins when it covers at least as many loops as
    // the vertical prefix (c5: [prim] [mass, mom x3, energy] [update, prim];
    // c2's 13-loop vertical fusion keeps its two short runs inside).
    const bool horiz_ok = horiz && choice.max_loops == 0 && choice.nt == 0;
    const size_t hend = horiz_ok ? horizontal_run(chain, begin, begin + static_cast<size_t>(hmaxl)) : begin;
    if (horiz_ok)
      for (size_t e = begin + 1; e < best_end; ++e) {
        const size_t re = horizontal_run(chain, e, e + static_cast<size_t>(hmaxl));
        if (re >= e + 3 && re > best_end) {
          best_end = e;
          break;
        }
      }
    const bool use_horizontal = horiz_ok && hend >= begin + 2 && hend - begin >= best_end - begin;
    // Horizontal run: independent loops over one range fused point by point.
    if (use_horizontal) {
      {
        const LoopChain sub = slice_chain(chain, begin, hend);
        StreamKernel K;
        K.begin = begin;
        K.end = hend;
        K.dim = chain.dim;
        std::map<DatasetId, int> slot;
        for (const LoopRecord& lp : sub.loops)
          for (const ArgSpec& a : lp.args)
            if (!slot.count(a.dataset)) {
              slot[a.dataset] = static_cast<int>(K.dats.size());
              K.dats.push_back(a.dataset);
            }
        const size_t nd = K.dats.size();
        K.load.assign(nd, 1);
        K.store.assign(nd, 0);
        K.pingpong.assign(nd, 0);
        K.store_box.assign(nd, Range(chain.dim));
        for (const LoopRecord& lp : sub.loops)
          for (const ArgSpec& a : lp.args)
            if (mode_writes(a.mode)) {
              K.store[static_cast<size_t>(slot[a.dataset])] = 1;
              K.store_box[static_cast<size_t>(slot[a.dataset])] = lp.range;
            }
        int np = 0;
        for (const LoopRecord& lp : sub.loops) {
          K.param_off.push_back(np);
          np += static_cast<int>(lp.kernel.fn.params.size());
        }
        K.nparams = np;
        for (const LoopRecord& lp : sub.loops) K.recorded_points += lp.range.volume();
        K.computed_points = K.recorded_points;
        K.live_loops = static_cast<int>(sub.size());
        K.hull = sub.loops[0].range;
        for (size_t li = 0; li < sub.size(); ++li) {
          K.loop_range.push_back(sub.loops[li].range);
          K.loop_live.push_back(1);
          K.loop_need.push_back(std::array<int64_t, 6>{0, 0, 0, 0, 0, 0});
        }
        const int ntx = chain.dim == 3 ? env_int("TCG_STREAM_HNTX", 64) : 128;
        const int nty = chain.dim == 3 ? env_int("TCG_STREAM_HNTY", 2) : 1;
        // Measured on c5 (profiles/r5/sweeps.md): 64 x 2 threads; 2 planes per thread 190 ms/step,
        // 1 plane 202, 3 planes 195, 4 planes 210, 8 planes 209 (registers); 32 x 4 threads 188, 64 x 4 247.
        const int run = env_int("TCG_STREAM_HRUN", 2);
        K.source = generate_horizontal(sub, geoms, K.param_off, np, K, ntx, nty, run, red_mask);
        K.tile_points = static_cast<int64_t>(K.nt) * run;
        K.warm_rows = 0;
        K.hash = fnv(K.source);
        plan.kernels.push_back(std::move(K));
        begin = hend;
        continue;
      }
    }
    const size_t end = best_end;
    const LoopChain sub = slice_chain(chain, begin, end);
    const Analysis A = analyze(sub, nostore_at(begin, end));
    StreamKernel K;
    K.begin = begin;
    K.end = end;
    K.dim = chain.dim;
    K.dats = A.dats;
    const size_t nd = A.dats.size();
    K.load.assign(nd, 0);
    K.store.assign(nd, 0);
    K.pingpong.assign(nd, 0);
    K.store_box.assign(nd, Range(chain.dim));
    for (size_t k = 0; k < nd; ++k) {
      const int iv = A.input_ver[k];
      K.load[k] = iv >= 0 && A.vers[static_cast<size_t>(iv)].needed;
      if (A.final_ver[k] >= 0 && A.vers[static_cast<size_t>(A.final_ver[k])].store) {
        K.store[k] = 1;
        K.store_box[k] = A.whull[k];
        // In place is safe only when no CTA can read the dataset's starting
        // state at a point some CTA overwrites: the input is read only to
        // pass through points outside the first writer's range, and every
        // later writer stays inside that range.
        const bool inplace = iv < 0 || !A.vers[static_cast<size_t>(iv)].needed ||
                             (A.vers[static_cast<size_t>(iv)].pass_only && A.all_w_in_first[k]);
        K.pingpong[k] = inplace ? 0 : 1;
      }
    }
    int np = 0;
    for (const LoopRecord& lp : sub.loops) {
      K.param_off.push_back(np);
      np += static_cast<int>(lp.kernel.fn.params.size());
    }
    K.nparams = np;
    if (!A.any_out) {
      K.nt = 32;
      K.nctas = 0;
      plan.kernels.push_back(K);
      begin = end;
      continue;
    }
    Sched sc;
    const Shape S = size_kernel(A, sub, dev, choice, sc);
    K.nt = S.nt;
    K.minb = S.minb;
    K.bx = S.blk.bx;
    K.by = S.blk.by;
    K.ntx = S.ntx;
    K.smem_bytes = static_cast<int>(S.smem_bytes);
    K.nctas = S.nxt * S.nyt * S.ns;
    K.tile[0] = S.tx;
    K.tile[1] = S.ty;
    K.owned[0] = static_cast<int>(S.wox);
    K.owned[1] = static_cast<int>(S.woy);
    K.grid[0] = static_cast<int>(S.nxt);
    K.grid[1] = static_cast<int>(S.nyt);
    K.grid[2] = static_cast<int>(S.ns);
    for (int d = 0; d < 3; ++d)
      for (int e = 0; e < 2; ++e) K.ext[d][e] = A.E[d][e];
    K.lag_max = static_cast<int>(sc.lmax);
    K.ring_doubles = sc.reg_doubles;
    K.smem_stages = sc.smem_rows;
    int nloops_live = 0;
    for (size_t li = 0; li < sub.size(); ++li) {
      K.recorded_points += sub.loops[li].range.volume();
      nloops_live += A.loops[li].needed ? 1 : 0;
    }
    K.hull = A.H;
    for (size_t li = 0; li < sub.size(); ++li) {
      K.loop_range.push_back(sub.loops[li].range);
      K.loop_live.push_back(A.loops[li].needed ? 1 : 0);
      std::array<int64_t, 6> nd6{0, 0, 0, 0, 0, 0};
      for (int d = 0; d < A.dim; ++d)
        for (int e = 0; e < 2; ++e) nd6[static_cast<size_t>(2 * d + e)] = std::max<int64_t>(0, A.loops[li].need[d][e]);
      K.loop_need.push_back(nd6);
    }
    K.tiles = S.nxt * S.nyt;
    K.stream_extent = A.H.extent(A.s);
    K.warm_rows = A.E[A.s][0] + A.E[A.s][1] + sc.lmax;
    // Shortest segment = TCG_STREAM_MIN_SEG_WARM x the pipeline warm-up. It only binds when the tiles
    // underfill the GPU (c1: 9 tiles on 592 slots). Measured on c1 (profiles/r5/sweeps.md): 4x warm-up
    // 0.0539 ms/chain (99 + 207 CTAs), 3x 0.0454, 2x 0.0394, 1x 0.0365 (1233 CTAs) -- short segments
    // recompute more rows but every CTA walks fewer steps; c2 / c4 (slots already full) are unaffected.
    K.min_seg = std::max<int64_t>(8, static_cast<int64_t>(env_dbl("TCG_STREAM_MIN_SEG_WARM", 1.0) * static_cast<double>(K.warm_rows)));
    K.tile_points = static_cast<int64_t>(S.tx) * S.ty;
    K.live_loops = nloops_live;
    K.forced_segments = choice.segments;
    K.computed_points = K.computed_for(S.ns);
    K.source = generate(sub, A, sc, S, geoms, red_mask, K.param_off, np, K);
    K.hash = fnv(K.source);
    plan.kernels.push_back(std::move(K));
    begin = end;
  }
  plan.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return plan;
}

}  // namespace tcg
