// hetbridge — static race and bounds check of a launch's device tables.
//
// The pool's compute-sanitizer is closed (runs under it left GPUs needing a
// reset), and racecheck would only see shared memory anyway. The hazards of
// these kernels are global-memory ones, and every global address a boundary
// kernel touches comes from the descriptor tables this runtime uploads. So the
// tables themselves are checked, as the kernels will read them (downloaded
// back from the device), for every buffer set:
//   bounds   every copy source / destination run, every reduce term and
//            accumulator lies inside one planned buffer of the right slot and
//            buffer set (strided buffers: inside one row), gather id arrays
//            inside the TEXT buffer;
//   ownership pull mode writes only this GPU's destinations, push mode reads
//            only this GPU's sources, the gradient return writes only this
//            GPU's accumulators;
//   races    no two destination runs of a launch overlap (write/write across
//            CTAs), no source run overlaps a destination (read/write), no two
//            accumulators overlap, no term overlaps an accumulator;
//   protocol every run that touches a peer's buffer sits in the remote queue,
//            i.e. behind the in-kernel peer wait (a local-queue chunk starts
//            before the peers have arrived: reading a peer there would be a
//            race with the peer's producer), and its `peers` mask names them;
//   coverage every chunk of every segment is handed out exactly once.
// The device analogue for the cross-GPU order is the out-of-turn check in the
// kernels (launch_protocol.cuh spin_until, R:core/src/simnet.cpp:202-207).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "hb/error.hpp"
#include "hb/runtime.hpp"

namespace hb::rt {

namespace {

struct DeviceGuard {  // the exec's device current for the scope
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct Extent {
  uintptr_t lo = 0, hi = 0;  // [lo, hi)
  int rank = -1, slot = -1;
  uint64_t row_bytes = 0, stride_bytes = 0;  // stride_bytes 0: packed
};

struct Iv {
  uintptr_t lo, hi;
  const char* what;
  size_t seg;
};

template <class T>
std::vector<T> download(const T* p, size_t n) {
  std::vector<T> v(n);
  if (n) {
    const cudaError_t e = cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) raise(ErrorCode::CudaError, std::string("validate: download: ") + cudaGetErrorString(e));
  }
  return v;
}

std::string hex(uintptr_t p) {
  char b[32];
  std::snprintf(b, sizeof b, "0x%llx", static_cast<unsigned long long>(p));
  return b;
}

// Whether two intervals of `a` overlap (sorted in place); *why names the first pair.
bool first_overlap(std::vector<Iv>& a, std::string* why) {
  std::sort(a.begin(), a.end(), [](const Iv& x, const Iv& y) { return x.lo < y.lo; });
  for (size_t i = 1; i < a.size(); ++i)
    if (a[i].lo < a[i - 1].hi) {
      *why = std::string(a[i - 1].what) + " of segment " + std::to_string(a[i - 1].seg) + " [" + hex(a[i - 1].lo) +
             "," + hex(a[i - 1].hi) + ") overlaps " + a[i].what + " of segment " + std::to_string(a[i].seg) + " [" +
             hex(a[i].lo) + "," + hex(a[i].hi) + ")";
      return true;
    }
  return false;
}

// Any interval of `r` that intersects one of `w` (both sorted by lo).
bool cross_overlap(std::vector<Iv>& r, std::vector<Iv>& w, std::string* why) {
  std::sort(r.begin(), r.end(), [](const Iv& x, const Iv& y) { return x.lo < y.lo; });
  std::sort(w.begin(), w.end(), [](const Iv& x, const Iv& y) { return x.lo < y.lo; });
  size_t j = 0;
  for (const auto& x : r) {
    while (j < w.size() && w[j].hi <= x.lo) ++j;
    for (size_t k = j; k < w.size() && w[k].lo < x.hi; ++k)
      if (w[k].hi > x.lo) {
        *why = std::string(x.what) + " of segment " + std::to_string(x.seg) + " overlaps " + w[k].what +
               " of segment " + std::to_string(w[k].seg);
        return true;
      }
  }
  return false;
}

}  // namespace

std::string Exec::validate(uint64_t* checks) {
  DeviceGuard dg(device_);
  prepare_fwd();
  prepare_bwd();
  uint64_t n = 0;
  std::string why;
  auto fail = [&](const std::string& m) {
    if (why.empty()) why = m;
  };

  for (int mb = 0; mb < cfg_.mb_slots && why.empty(); ++mb) {
    // planned buffers of this buffer set whose address this GPU can resolve
    std::vector<Extent> ext;
    for (int r = 0; r < map_.world; ++r)
      for (int s = 0; s < index::kNumSlots; ++s) {
        if (!map_.elems[r][s]) continue;
        const int es = s == index::kText && cfg_.text_embedding ? 4 : dev::dtype_size(slot_dtype(s));
        unsigned char* p = nullptr;
        try {
          p = addr(r, s, mb, 0, es);
        } catch (const Error&) {
          continue;  // a peer's buffer this GPU never opened (not in its work)
        }
        Extent e;
        e.rank = r;
        e.slot = s;
        const int64_t w = s == index::kText && cfg_.text_embedding ? 1 : row_width(s);
        e.row_bytes = static_cast<uint64_t>(w) * es;
        const Binding* b = binding_of(r, s, mb);
        const uint64_t rows = static_cast<uint64_t>(map_.elems[r][s] / (s == index::kText && cfg_.text_embedding
                                                                             ? splice_d_h_ : w));
        if (b && b->stride) {
          e.stride_bytes = static_cast<uint64_t>(b->stride) * es;
          e.lo = reinterpret_cast<uintptr_t>(p);
          e.hi = e.lo + (rows - 1) * e.stride_bytes + e.row_bytes;
        } else {
          e.lo = reinterpret_cast<uintptr_t>(p);
          e.hi = e.lo + slot_bytes(r, s);
        }
        ext.push_back(e);
      }
    // the extent holding [lo, hi) of one of `slots`, or nullptr
    auto find = [&](uintptr_t lo, uintptr_t hi, std::initializer_list<int> slots) -> const Extent* {
      for (const auto& e : ext) {
        if (std::find(slots.begin(), slots.end(), e.slot) == slots.end()) continue;
        if (lo < e.lo || hi > e.hi) continue;
        if (e.stride_bytes) {  // a strided buffer: the run must stay inside one row
          const uint64_t o = (lo - e.lo) % e.stride_bytes;
          if (o + (hi - lo) > e.row_bytes) continue;
        }
        return &e;
      }
      return nullptr;
    };
    const std::string at = " (buffer set " + std::to_string(mb) + ")";

    // ---- forward: copy table
    std::vector<Iv> writes, reads;
    const auto cs = download(tables_[mb].copy, fwd_local_.size());
    for (size_t i = 0; i < cs.size(); ++i) {
      const auto& c = cs[i];
      ++n;
      if (c.ndst < 1 || c.ndst > dev::kMaxFan) fail("copy segment " + std::to_string(i) + ": bad fan " + std::to_string(c.ndst));
      const uintptr_t s0 = reinterpret_cast<uintptr_t>(c.src);
      bool touches_peer = false;
      if (c.ids) {  // gather run: ids in TEXT, rows from the embedding table
        const uint64_t rows = c.row_bytes ? c.nbytes / c.row_bytes : 0;
        const uintptr_t i0 = reinterpret_cast<uintptr_t>(c.ids);
        const Extent* e = find(i0, i0 + rows * 4, {index::kText});
        if (!e || c.row_bytes == 0 || rows * c.row_bytes != c.nbytes ||
            (c.shards ? c.shard_rows == 0 : s0 != reinterpret_cast<uintptr_t>(embed_table_)))
          fail("copy segment " + std::to_string(i) + ": gather ids/table out of bounds" + at);
        else if (gpu_of(e->rank) != my_gpu_) touches_peer = true;
        reads.push_back({i0, i0 + rows * 4, "gather ids", i});
        if (c.shards) {  // vocab-parallel: every shard base is a known rank's shard; peers' behind the wait
          const auto sp = download(c.shards, static_cast<size_t>(plan_.edge.dest.tp));
          for (const unsigned char* p : sp) {
            int owner = -1;
            for (int r = 0; r < map_.world && owner < 0; ++r)
              if (shard_of(r).ptr == p) owner = r;
            if (owner < 0) {
              fail("copy segment " + std::to_string(i) + ": gather shard base is no rank's embedding shard");
            } else if (gpu_of(owner) != my_gpu_) {
              touches_peer = true;
              if (!((c.peers >> gpu_of(owner)) & 1u))
                fail("copy segment " + std::to_string(i) + ": peers mask misses shard GPU " + std::to_string(gpu_of(owner)));
            }
          }
        }
      } else {
        const Extent* e = find(s0, s0 + c.nbytes, {index::kSrcAct, index::kText});
        if (!e) {
          fail("copy segment " + std::to_string(i) + ": source run [" + hex(s0) + ", +" + std::to_string(c.nbytes) +
               ") outside every source buffer" + at);
        } else {
          if (gpu_of(e->rank) != my_gpu_) {
            touches_peer = true;
            if (fwd_push_) fail("copy segment " + std::to_string(i) + ": push mode reads a peer's source" + at);
            if (!((c.peers >> gpu_of(e->rank)) & 1u))
              fail("copy segment " + std::to_string(i) + ": peers mask misses source GPU " + std::to_string(gpu_of(e->rank)));
          }
        }
        reads.push_back({s0, s0 + c.nbytes, "source run", i});
      }
      for (int d = 0; d < c.ndst && d < dev::kMaxFan; ++d) {
        ++n;
        const uintptr_t d0 = reinterpret_cast<uintptr_t>(c.dst[d]);
        const Extent* e = find(d0, d0 + c.nbytes, {index::kDstAct});
        if (!e) {
          fail("copy segment " + std::to_string(i) + ": destination " + std::to_string(d) + " outside every "
               "destination buffer" + at);
        } else if (gpu_of(e->rank) != my_gpu_) {
          touches_peer = true;
          if (!fwd_push_) fail("copy segment " + std::to_string(i) + ": pull mode writes a peer's destination" + at);
          if (!((c.peers >> gpu_of(e->rank)) & 1u))
            fail("copy segment " + std::to_string(i) + ": peers mask misses destination GPU " + std::to_string(gpu_of(e->rank)));
        }
        writes.push_back({d0, d0 + c.nbytes, "destination run", i});
      }
      if (touches_peer != static_cast<bool>(fwd_local_[i].remote))
        fail("copy segment " + std::to_string(i) + (touches_peer ? ": touches a peer but is in the local queue"
                                                                 : ": local but in the remote queue"));
    }
    if (why.empty() && first_overlap(writes, &why)) why = "forward write/write race: " + why + at;
    if (why.empty() && cross_overlap(reads, writes, &why)) why = "forward read/write race: " + why + at;
    n += writes.size() + reads.size();

    // ---- backward: reduce table and side array
    const auto rs = download(tables_[mb].reduce, static_cast<size_t>(bwd_groups_));
    size_t nside = 0;
    for (const auto& r : rs)
      nside = std::max<size_t>(nside, std::max<size_t>(static_cast<size_t>(r.term0 + r.nterms), static_cast<size_t>(r.dst0 + r.ndst)));
    const auto side = download(reinterpret_cast<const uintptr_t*>(tables_[mb].terms), nside);
    const int es_in = dev::dtype_size(cfg_.grad_in_dtype), es_out = dev::dtype_size(cfg_.grad_out_dtype);
    std::vector<Iv> accs, terms;
    for (size_t i = 0; i < rs.size(); ++i) {
      const auto& r = rs[i];
      ++n;
      if (r.nterms < 1 || r.ndst < 1 || r.ndst > dev::kMaxFan || r.term0 < 0 || r.dst0 < 0) {
        fail("reduce segment " + std::to_string(i) + ": bad term/accumulator counts");
        continue;
      }
      if (side[r.dst0] != reinterpret_cast<uintptr_t>(r.dst))
        fail("reduce segment " + std::to_string(i) + ": dst differs from its first accumulator");
      uint32_t peers = 0;
      for (int t = 0; t < r.nterms; ++t) {
        ++n;
        const uintptr_t p = side[r.term0 + t];
        const Extent* e = find(p, p + r.nelem * es_in, {index::kDstGrad});
        if (!e) fail("reduce segment " + std::to_string(i) + ": term " + std::to_string(t) + " outside every gradient buffer" + at);
        else if (gpu_of(e->rank) != my_gpu_) peers |= 1u << gpu_of(e->rank);
        terms.push_back({p, p + r.nelem * es_in, "term", i});
      }
      if ((peers & ~r.peers) != 0) fail("reduce segment " + std::to_string(i) + ": peers mask misses a term's GPU");
      for (int d = 0; d < r.ndst; ++d) {
        ++n;
        const uintptr_t p = side[r.dst0 + d];
        const Extent* e = find(p, p + r.nelem * es_out, {index::kSrcGrad});
        if (!e) fail("reduce segment " + std::to_string(i) + ": accumulator " + std::to_string(d) + " outside every source-gradient buffer" + at);
        else if (gpu_of(e->rank) != my_gpu_) fail("reduce segment " + std::to_string(i) + ": writes a peer's accumulator" + at);
        accs.push_back({p, p + r.nelem * es_out, "accumulator", i});
      }
    }
    if (why.empty() && first_overlap(accs, &why)) why = "backward write/write race: " + why + at;
    if (why.empty() && cross_overlap(terms, accs, &why)) why = "backward read/write race: " + why + at;
    n += accs.size() + terms.size();

    // ---- protocol and coverage of the hand-out tables (chunks are shared by every buffer set)
    if (mb == 0 && why.empty()) {
      auto cover = [&](const DevPartition& P, size_t nseg, auto len_of, auto remote_of, const char* dir) {
        if (P.mode != dev::kPartDynamic && P.mode != dev::kPartTma) return;
        const auto lq = download(P.chunks, P.total_chunks);
        const auto rq = download(P.rchunks, P.rtotal_chunks);
        std::vector<std::vector<uint32_t>> seen(nseg);
        for (int q = 0; q < 2; ++q)
          for (const auto& c : q ? rq : lq) {
            ++n;
            if (c.x >= nseg) {
              fail(std::string(dir) + ": chunk names segment " + std::to_string(c.x) + " of " + std::to_string(nseg));
              return;
            }
            if (remote_of(c.x) && q == 0)
              fail(std::string(dir) + " segment " + std::to_string(c.x) + " touches a peer but is handed out "
                   "before the peer wait (local queue)");
            for (uint32_t u = 0; u <= (c.y >> 24); ++u) seen[c.x].push_back((c.y & 0xffffffu) + u);
          }
        for (size_t s = 0; s < nseg; ++s) {
          const uint64_t u = remote_of(s) ? P.rchunk : P.chunk;
          const uint64_t k = (len_of(s) + u - 1) / u;
          auto& v = seen[s];
          std::sort(v.begin(), v.end());
          bool ok = v.size() == k;
          for (size_t j = 0; ok && j < v.size(); ++j) ok = v[j] == j;
          if (!ok) fail(std::string(dir) + " segment " + std::to_string(s) + ": chunks not handed out exactly once");
        }
      };
      cover(fwd_part_, cs.size(), [&](size_t s) { return cs[s].nbytes; },
            [&](size_t s) { return static_cast<bool>(fwd_local_[s].remote); }, "forward");
      cover(bwd_part_, rs.size(), [&](size_t s) { return rs[s].nelem; },
            [&](size_t s) { return rs[s].peers != 0; }, "backward");
    }
  }
  if (checks) *checks = n;
  return why;
}

}  // namespace hb::rt
