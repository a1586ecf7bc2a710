// fft_host.cu -- host-side FFT planning: factorisation and twiddle tables (long double).
#include <cmath>

#include "fft.cuh"

namespace se1p {

bool fft_factor(int n, std::vector<int>& rad, bool r8) {
  rad.clear();
  if (n < 1) return false;
  // odd radices first: the first stage writes with stride R, conflict-free in shared memory
  // when R is odd; then 8s (fewest shared-memory passes), 4, 2
  int m = n;
  std::vector<int> odd, even;
  while (r8 && m % 9 == 0) { odd.push_back(9); m /= 9; }
  while (m % 3 == 0) { odd.push_back(3); m /= 3; }
  while (m % 5 == 0) { odd.push_back(5); m /= 5; }
  while (r8 && m % 8 == 0) { even.push_back(8); m /= 8; }
  while (m % 4 == 0) { even.push_back(4); m /= 4; }
  while (m % 2 == 0) { even.push_back(2); m /= 2; }
  rad = odd;
  rad.insert(rad.end(), even.begin(), even.end());
  for (int p = 7; m > 1; p += 2) {
    while (m % p == 0) {
      if (p > kMaxGenericRadix) return false;
      rad.push_back(p);
      m /= p;
    }
    if (p > kMaxGenericRadix && m > 1) return false;
  }
  return (int)rad.size() <= kMaxStages;
}

static double2 unit_root(long long num, long long den) {
  // e^{-2 pi i num/den}, with num reduced mod den first (exact) and long double trig
  long long r = num % den;
  if (r < 0) r += den;
  const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)r / (long double)den;
  return make_double2((double)cosl(a), (double)sinl(a));
}

bool fft_make(int n, FftDesc& d, std::vector<double2>& table, bool r8) {
  std::vector<int> rad;
  if (!fft_factor(n, rad, r8)) return false;
  d.n = n;
  d.nst = (int)rad.size();
  int Ns = 1;
  for (int s = 0; s < d.nst; ++s) {
    const int R = rad[s];
    d.rad[s] = R;
    d.twoff[s] = (int)table.size();
    for (int k = 0; k < Ns; ++k)
      for (int t = 1; t < R; ++t) table.push_back(unit_root((long long)t * k, (long long)Ns * R));
    d.rootoff[s] = (int)table.size();
    if (R != 2 && R != 3 && R != 4 && R != 5 && R != 8 && R != 9)
      for (int k = 0; k < R; ++k) table.push_back(unit_root(k, R));
    Ns *= R;
  }
  d.total = (int)table.size();
  return true;
}

bool fft_friendly(int n) {
  if (n < 1) return false;
  for (int p : {2, 3, 5})
    while (n % p == 0) n /= p;
  return n == 1;
}

// Smallest n' >= n whose factors are 2, 3, 5: every stage then has a dedicated butterfly.
int next_friendly(int n) {
  while (!fft_friendly(n)) ++n;
  return n;
}

}  // namespace se1p
