// records.h -- host-side dataset writer: CSR shot records -> records.jsonl text.
//
// Restates the reference's record emission (ref execute.py:181-223 sorts each
// trajectory's counts by bitstring; execute.py:246-259 writes one
// json.dumps({"t","b","c"}, separators=(",", ":")) line per record;
// statevector.py:44-53 formats basis index v as format(v, "0{n}b"), qubit n-1
// leftmost) straight from the sampler's packed output, so a 10^8-record
// config-4 dataset is formatted at memory speed on all host cores instead of
// one json.dumps call per record.
//
// Layout: trajectory i owns records [offsets[i], offsets[i+1]) of
// indices/counts and is written with id traj_ids[i].  Fixed-width binary
// strings order like their integers, so "sorted by bitstring" is "sorted by
// index"; segments the sampler did not emit ascending are sorted on a copy.
// Two phases: per-trajectory byte sizes (exact, from digit counts) -> prefix
// sum -> every thread formats its own contiguous trajectory range in place.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <utility>
#include <vector>

namespace ptsbe_records {

inline int dec_len(uint64_t v) {
  int d = 1;
  while (v >= 10) { v /= 10; ++d; }
  return d;
}

inline char* put_dec(char* p, uint64_t v) {
  char tmp[24];
  int k = 0;
  do { tmp[k++] = char('0' + v % 10); v /= 10; } while (v);
  while (k) *p++ = tmp[--k];
  return p;
}

// {"t":  ,"b":"  ","c":  }\n  -> 5 + 6 + 6 + 2 fixed bytes
constexpr int64_t kFixed = 19;

// byte value -> its 8 binary digits, most significant first
struct BitChars {
  char c[256][8];
  BitChars() {
    for (int b = 0; b < 256; ++b)
      for (int j = 0; j < 8; ++j) c[b][j] = char('0' + ((b >> (7 - j)) & 1));
  }
};

inline char* put_bits(char* p, int n, uint64_t v) {
  static const BitChars tbl;
  int j = n - 1;
  for (; (j + 1) & 7; --j) *p++ = char('0' + ((v >> j) & 1u));   // leading n % 8 bits
  for (; j >= 0; j -= 8) { std::memcpy(p, tbl.c[(v >> (j - 7)) & 0xff], 8); p += 8; }
  return p;
}

inline char* put_record(char* p, uint64_t t, int n, uint64_t v, uint64_t c) {
  std::memcpy(p, "{\"t\":", 5); p += 5;
  p = put_dec(p, t);
  std::memcpy(p, ",\"b\":\"", 6); p += 6;
  p = put_bits(p, n, v);
  std::memcpy(p, "\",\"c\":", 6); p += 6;
  p = put_dec(p, c);
  *p++ = '}';
  *p++ = '\n';
  return p;
}

inline bool ascending(const uint64_t* idx, int64_t lo, int64_t hi) {
  for (int64_t i = lo + 1; i < hi; ++i)
    if (idx[i - 1] >= idx[i]) return false;
  return true;
}

// Returns the total byte length; formats into buf when buf != nullptr and
// cap >= that length; -1 on invalid arguments.
inline int64_t format(int n, int64_t n_traj, const int64_t* ids, const int64_t* off,
                      const uint64_t* idx, const uint32_t* cnt, char* buf, int64_t cap) {
  if (n < 1 || n > 64 || n_traj < 0 || (n_traj > 0 && (!ids || !off))) return -1;
  if (n_traj > 0 && off[0] < 0) return -1;
  for (int64_t i = 0; i < n_traj; ++i) {
    if (off[i + 1] < off[i] || ids[i] < 0) return -1;
  }
  const int64_t n_rec = n_traj > 0 ? off[n_traj] - off[0] : 0;
  if (n_rec > 0 && (!idx || !cnt)) return -1;
  if (n < 64) {
    for (int64_t r = n_traj > 0 ? off[0] : 0; r < (n_traj > 0 ? off[n_traj] : 0); ++r)
      if (idx[r] >> n) return -1;
  }

  unsigned hw = std::thread::hardware_concurrency();
  int nth = (int)std::max(1u, std::min(hw ? hw : 1u, 64u));
  if (n_rec < (1 << 16)) nth = 1;

  // phase 1: bytes per trajectory
  std::vector<int64_t> pos(n_traj + 1, 0);
  auto size_range = [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      int64_t s = 0;
      const int64_t per = kFixed + n + dec_len((uint64_t)ids[i]);
      for (int64_t r = off[i]; r < off[i + 1]; ++r) s += per + dec_len(cnt[r]);
      pos[i + 1] = s;
    }
  };
  auto parallel = [&](auto&& fn) {
    if (nth == 1) { fn(0, n_traj); return; }
    std::vector<std::thread> th;
    // split by record count so threads get equal work
    int64_t lo_t = 0;
    const int64_t base = off[0];
    for (int k = 0; k < nth && lo_t < n_traj; ++k) {
      const int64_t goal = base + n_rec * (k + 1) / nth;
      int64_t hi_t = lo_t;
      while (hi_t < n_traj && (off[hi_t + 1] <= goal || hi_t == lo_t)) ++hi_t;
      if (k == nth - 1) hi_t = n_traj;
      th.emplace_back(fn, lo_t, hi_t);
      lo_t = hi_t;
    }
    for (auto& t : th) t.join();
  };
  parallel(size_range);
  for (int64_t i = 0; i < n_traj; ++i) pos[i + 1] += pos[i];
  const int64_t total = pos[n_traj];
  if (!buf || cap < total) return total;

  // phase 2: format in place
  auto write_range = [&](int64_t a, int64_t b) {
    std::vector<std::pair<uint64_t, uint32_t>> tmp;
    for (int64_t i = a; i < b; ++i) {
      char* p = buf + pos[i];
      const uint64_t t = (uint64_t)ids[i];
      if (ascending(idx, off[i], off[i + 1])) {
        for (int64_t r = off[i]; r < off[i + 1]; ++r) p = put_record(p, t, n, idx[r], cnt[r]);
      } else {
        tmp.clear();
        for (int64_t r = off[i]; r < off[i + 1]; ++r) tmp.emplace_back(idx[r], cnt[r]);
        std::sort(tmp.begin(), tmp.end());
        for (auto& e : tmp) p = put_record(p, t, n, e.first, e.second);
      }
    }
  };
  parallel(write_range);
  return total;
}

}  // namespace ptsbe_records
