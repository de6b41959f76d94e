// vf_format.cpp -- host-side output formats:
// the feature lines of report.dump_features (/root/reference/pkg/src/vidfeat/
// report.py:102-113).  Python's f"{v:.4f}" and glibc's "%.4f" are both
// correctly rounded (round-half-even on the exact binary value), so the text is
// byte-identical.  Features are split across threads; each formats its range
// into its own buffer, then the pieces are concatenated in order.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/vidfeat_b200.h"

namespace {

// "%.{P}f" of v, correctly rounded (round half to even on the exact binary
// value, as Python's format() and glibc's printf).  v = M * 2^E exactly; the
// integer N = round(v * 10^P) comes from 128-bit arithmetic.  Returns the
// length written to buf, or -1 to fall back to snprintf (nan, inf, |v| large).
int fixed(double v, int P, char* buf)
{
  if (!std::isfinite(v) || std::fabs(v) >= 1e12) return -1;
  static const uint64_t pow10[] = {1, 10, 100, 1000, 10000, 100000, 1000000};
  int e2;
  const double fr = std::frexp(std::fabs(v), &e2);             // |v| = fr * 2^e2, fr in [0.5, 1)
  const uint64_t M = (uint64_t)std::ldexp(fr, 53);            // exact 53-bit integer
  const int E = e2 - 53;                                      // |v| = M * 2^E
  unsigned __int128 num = (unsigned __int128)M * pow10[P];
  uint64_t N;
  if (M == 0) {
    N = 0;
  } else if (E >= 0) {
    N = (uint64_t)(num << E);                                 // |v| < 1e12: fits
  } else {
    const int k = -E;
    if (k >= 127) {
      N = 0;                                                  // < 2^-54 * 10^P: rounds to 0
    } else {
      const unsigned __int128 q = num >> k, r = num & (((unsigned __int128)1 << k) - 1);
      const unsigned __int128 half = (unsigned __int128)1 << (k - 1);
      N = (uint64_t)q + ((r > half || (r == half && (q & 1))) ? 1 : 0);
    }
  }
  char tmp[32];
  int n = 0;
  do { tmp[n++] = (char)('0' + N % 10); N /= 10; } while (N);
  while (n < P + 1) tmp[n++] = '0';                           // at least "0.xxxx"
  int o = 0;
  if (std::signbit(v)) buf[o++] = '-';
  for (int i = n - 1; i >= P; i--) buf[o++] = tmp[i];
  buf[o++] = '.';
  for (int i = P - 1; i >= 0; i--) buf[o++] = tmp[i];
  return o;
}

int fmt(double v, int P, char* buf, size_t cap)
{
  const int n = fixed(v, P, buf);
  return n >= 0 ? n : snprintf(buf, cap, P == 4 ? "%.4f" : "%.6f", v);
}

void format_range(int64_t lo, int64_t hi, const double* x, const double* y, const double* sg, const double* th,
                  const uint8_t* org, const uint8_t* desc, std::string& out)
{
  static const char hexd[] = "0123456789abcdef";
  char num[4][64];
  out.clear();
  if (out.capacity() < (size_t)(hi - lo) * 200) out.reserve((size_t)(hi - lo) * 200);
  for (int64_t i = lo; i < hi; i++) {
    const int a = fmt(x[i], 4, num[0], sizeof(num[0]));
    const int b = fmt(y[i], 4, num[1], sizeof(num[1]));
    const int c = fmt(sg[i], 4, num[2], sizeof(num[2]));
    const int d = fmt(th[i], 6, num[3], sizeof(num[3]));
    out.append(num[0], a); out.push_back(' ');
    out.append(num[1], b); out.push_back(' ');
    out.append(num[2], c); out.push_back(' ');
    out.append(num[3], d); out.push_back(' ');
    out.append(org[i] ? "propagated" : "detected");
    out.push_back(' ');
    char hx[128];
    const uint8_t* p = desc + 64 * i;
    for (int k = 0; k < 64; k++) { hx[2 * k] = hexd[p[k] >> 4]; hx[2 * k + 1] = hexd[p[k] & 15]; }
    out.append(hx, 128);
    out.push_back('\n');
  }
}

// Persistent workers (created on first use), each with a reusable line buffer.
struct Pool {
  std::mutex m;
  std::condition_variable cv, done;
  std::vector<std::thread> th;
  std::vector<std::string> part;
  std::function<void(int)> job;
  int gen = 0, pending = 0, nwork = 0;
  bool stop = false;
  explicit Pool(int n) : part(n) {
    for (int i = 1; i < n; i++)
      th.emplace_back([this, i] {
        int seen = 0;
        for (;;) {
          std::unique_lock<std::mutex> lk(m);
          cv.wait(lk, [&] { return stop || gen != seen; });
          if (stop) return;
          seen = gen;
          const bool mine = i < nwork;
          lk.unlock();
          if (mine) job(i);
          lk.lock();
          if (--pending == 0) done.notify_one();
        }
      });
  }
  ~Pool() {
    { std::lock_guard<std::mutex> lk(m); stop = true; }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  // job(t) for t in [0, n): worker 0 is the caller
  void run(int n, std::function<void(int)> f) {
    {
      std::lock_guard<std::mutex> lk(m);
      job = std::move(f);
      nwork = n;
      pending = (int)th.size();
      gen++;
    }
    cv.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(m);
    done.wait(lk, [&] { return pending == 0; });
  }
};

Pool& pool()
{
  static Pool p((int)std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  return p;
}

}  // namespace

extern "C" int vf_format_features(int64_t n, const double* x, const double* y, const double* sigma,
                                  const double* theta, const uint8_t* origin, const uint8_t* desc64, char* out,
                                  int64_t cap, int64_t* len)
{
  if (!len || n < 0 || cap < 0) return VF_ERR_ARG;
  *len = 0;
  if (n == 0) return VF_OK;
  if (!x || !y || !sigma || !theta || !origin || !desc64) return VF_ERR_ARG;
  static std::mutex call;                     // one formatting call at a time uses the pool
  std::lock_guard<std::mutex> guard(call);
  Pool& P = pool();
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)P.part.size(), n / 2048 + 1));
  P.run(nt, [&](int t) {
    format_range(n * t / nt, n * (t + 1) / nt, x, y, sigma, theta, origin, desc64, P.part[t]);
  });
  int64_t total = 0;
  for (int t = 0; t < nt; t++) total += (int64_t)P.part[t].size();
  *len = total;
  if (total > cap || !out) return out ? VF_ERR_CAPACITY : (cap == 0 ? VF_ERR_CAPACITY : VF_ERR_ARG);
  std::vector<int64_t> off(nt + 1, 0);
  for (int t = 0; t < nt; t++) off[t + 1] = off[t] + (int64_t)P.part[t].size();
  P.run(nt, [&](int t) { memcpy(out + off[t], P.part[t].data(), P.part[t].size()); });
  return VF_OK;
}
