// Python float repr for the trajectory log (host C++).
//
// The drop-in writes the reference's `episode_step` events (tuner.py:
// 414-420): json.dumps(sort_keys=True) of a dict whose "rewards" list holds
// every visited candidate's reward (P floats per step).  json renders each
// float with float.__repr__: the shortest digit string that round-trips
// (David Gay's dtoa mode 0), printed fixed when the decimal exponent is in
// (-4, 16] and as d.ddde+XX otherwise, with ".0" added to integral values;
// NaN / Infinity / -Infinity for the non-finite ones.  std::to_chars (C++17,
// libstdc++'s Ryu) yields the same shortest, nearest digits; this file
// formats them by CPython's rules (Python/pystrtod.c, format_float_short),
// splitting the list over worker threads.  Output is byte-identical to
// ", ".join(json's float repr) -- tests/test_repr_format.py checks millions of
// values, edge cases included, against json.dumps itself.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// one value into dst (>= 32 bytes available); returns bytes written
int repr_one(double x, char* dst) {
  if (std::isnan(x)) {
    memcpy(dst, "NaN", 3);
    return 3;
  }
  if (std::isinf(x)) {
    if (x > 0) {
      memcpy(dst, "Infinity", 8);
      return 8;
    }
    memcpy(dst, "-Infinity", 9);
    return 9;
  }
  char* p = dst;
  if (std::signbit(x)) {
    *p++ = '-';
    x = -x;
  }
  if (x == 0.0) {
    memcpy(p, "0.0", 3);
    return (int)(p - dst) + 3;
  }
  // shortest digits in scientific form: d[.ddd]e(+|-)XX
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci), x,
                               std::chars_format::scientific);
  const int len = (int)(r.ptr - sci);
  char digits[24];
  int nd = 0, i = 0;
  for (; i < len && sci[i] != 'e'; ++i)
    if (sci[i] != '.') digits[nd++] = sci[i];
  int e = 0;
  bool neg = false;
  ++i;  // 'e'
  if (sci[i] == '-') neg = true;
  ++i;
  for (; i < len; ++i) e = e * 10 + (sci[i] - '0');
  if (neg) e = -e;
  const int decpt = e + 1;   // value = 0.d1d2... x 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *p++ = digits[0];
    if (nd > 1) {
      *p++ = '.';
      memcpy(p, digits + 1, nd - 1);
      p += nd - 1;
    }
    *p++ = 'e';
    const int ex = decpt - 1;
    *p++ = ex < 0 ? '-' : '+';
    const int a = ex < 0 ? -ex : ex;
    if (a >= 100) {
      *p++ = (char)('0' + a / 100);
      *p++ = (char)('0' + (a / 10) % 10);
      *p++ = (char)('0' + a % 10);
    } else {
      *p++ = (char)('0' + a / 10);
      *p++ = (char)('0' + a % 10);
    }
  } else if (decpt <= 0) {
    *p++ = '0';
    *p++ = '.';
    for (int z = 0; z < -decpt; ++z) *p++ = '0';
    memcpy(p, digits, nd);
    p += nd;
  } else if (decpt >= nd) {
    memcpy(p, digits, nd);
    p += nd;
    for (int z = 0; z < decpt - nd; ++z) *p++ = '0';
    *p++ = '.';
    *p++ = '0';
  } else {
    memcpy(p, digits, decpt);
    p += decpt;
    *p++ = '.';
    memcpy(p, digits + decpt, nd - decpt);
    p += nd - decpt;
  }
  return (int)(p - dst);
}

}  // namespace

extern "C" {

// Python repr of v[0..n) joined by ", " (the body of json.dumps(list)) into
// out (cap bytes).  Returns the byte count, or -(bytes needed) when cap is
// too small (40 * n always suffices).  threads <= 0: hardware concurrency.
long long harl_format_floats(const double* v, long long n, char* out,
                             long long cap, int threads) {
  if (n <= 0) return 0;
  if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
  if (threads < 1) threads = 1;
  const long long per = 8192;
  long long chunks = (n + per - 1) / per;
  if (threads > chunks) threads = (int)chunks;
  // each chunk formats into its own buffer, then they are concatenated
  std::vector<std::vector<char>> bufs(chunks);
  auto work = [&](int tid) {
    for (long long c = tid; c < chunks; c += threads) {
      const long long a = c * per, b = a + per < n ? a + per : n;
      std::vector<char>& buf = bufs[c];
      buf.resize((size_t)(b - a) * 34);
      char* p = buf.data();
      for (long long k = a; k < b; ++k) {
        if (k > 0) {
          *p++ = ',';
          *p++ = ' ';
        }
        p += repr_one(v[k], p);
      }
      buf.resize((size_t)(p - buf.data()));
    }
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& t : pool) t.join();
  }
  long long total = 0;
  for (auto& b : bufs) total += (long long)b.size();
  if (total > cap) return -total;
  char* p = out;
  for (auto& b : bufs) {
    memcpy(p, b.data(), b.size());
    p += b.size();
  }
  return total;
}

// GBT refit output (heap layout: children of k at 2k+1, 2k+2; feat -2 = no
// node, -1 = leaf) -> _fit_tree's node numbering (costmodel.py:86-141: an
// explicit stack, left child first, both children allocated when the parent
// splits).  Per tree t: out_* [t][K] with the reference arrays in their
// first sizes[t] entries.
int harl_heap_to_creation_order(const int32_t* feat_h, const double* thr_h,
                                const double* val_h, int K, int n_trees,
                                int64_t* feature, double* threshold,
                                int64_t* left, int64_t* right, double* value,
                                int32_t* sizes) {
  if (!feat_h || !thr_h || !val_h || K < 1 || n_trees < 0 || !feature ||
      !threshold || !left || !right || !value || !sizes)
    return -1;
  std::vector<int> stack, ref(K);
  for (int t = 0; t < n_trees; ++t) {
    const int32_t* fh = feat_h + (size_t)t * K;
    const double* th = thr_h + (size_t)t * K;
    const double* vh = val_h + (size_t)t * K;
    int64_t* fo = feature + (size_t)t * K;
    double* to = threshold + (size_t)t * K;
    int64_t* lo = left + (size_t)t * K;
    int64_t* ro = right + (size_t)t * K;
    double* vo = value + (size_t)t * K;
    int n = 1;
    fo[0] = -1; to[0] = 0.0; lo[0] = -1; ro[0] = -1; vo[0] = 0.0;
    ref[0] = 0;
    stack.assign(1, 0);
    while (!stack.empty()) {
      const int h = stack.back();
      stack.pop_back();
      const int nid = ref[h];
      vo[nid] = vh[h];
      if (fh[h] < 0) continue;
      if (2 * h + 2 >= K) return -2;
      const int lid = n, rid = n + 1;
      n += 2;
      for (int c = lid; c <= rid; ++c) {
        fo[c] = -1; to[c] = 0.0; lo[c] = -1; ro[c] = -1; vo[c] = 0.0;
      }
      ref[2 * h + 1] = lid;
      ref[2 * h + 2] = rid;
      fo[nid] = fh[h];
      to[nid] = th[h];
      lo[nid] = lid;
      ro[nid] = rid;
      stack.push_back(2 * h + 2);
      stack.push_back(2 * h + 1);
    }
    sizes[t] = n;
  }
  return 0;
}

// ScheduleState.canonical (schedspace.py:117-120) of n states (tiles
// [n][slots] u16 with `levels` factors per tiled dim, knobs [n][3] u8):
// "<prefix>|t=a.b.c;d.e.f|ca=..|par=..|ur=.." per state, each followed by
// a NUL.  Returns the bytes written, or -(bytes needed) if cap is too small.
long long harl_format_canonical(const uint16_t* tiles, const uint8_t* knobs,
                                long long n, int slots, int levels,
                                const char* prefix, long long prefix_len,
                                char* out, long long cap) {
  if (n < 0 || slots < 0 || (slots && levels <= 0)) return 0;
  const long long per = prefix_len + 3 + 6LL * slots + 3 * (5 + 4 + 4) + 1;
  if (per * n > cap) return -(per * n);
  char* p = out;
  auto num = [&](unsigned v) {
    char b[8];
    int k = 0;
    do {
      b[k++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    while (k) *p++ = b[--k];
  };
  for (long long i = 0; i < n; ++i) {
    memcpy(p, prefix, (size_t)prefix_len);
    p += prefix_len;
    memcpy(p, "|t=", 3);
    p += 3;
    const uint16_t* t = tiles + i * slots;
    for (int s = 0; s < slots; ++s) {
      if (s) *p++ = (s % levels) ? '.' : ';';
      num(t[s]);
    }
    const uint8_t* k = knobs + i * 3;
    memcpy(p, "|ca=", 4);
    p += 4;
    num(k[0]);
    memcpy(p, "|par=", 5);
    p += 5;
    num(k[1]);
    memcpy(p, "|ur=", 4);
    p += 4;
    num(k[2]);
    *p++ = '\0';
  }
  return (long long)(p - out);
}

}  // extern "C"
