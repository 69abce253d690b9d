// Host write bandwidth probe: can 16 threads expand a run-length stream of
// labels into a 4 GB int32 image faster than PCIe delivers it (~55 GB/s)?
// g++ -O3 -march=native -pthread scripts/host_write_probe.cpp -o /tmp/hwp
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  const long long nv = 1000000000ll, row = 1000;
  const int T = argc > 1 ? atoi(argv[1]) : 16;
  int* img = (int*)aligned_alloc(64, nv * 4);
  std::memset(img, 0, nv * 4);  // pre-touch
  // runs: ~7 voxels mean (geometric), per row
  std::mt19937_64 rng(1);
  std::vector<int> lab;
  std::vector<unsigned short> start;
  std::vector<long long> roff(nv / row + 1);
  const long long nrows_sample = 20000;  // reuse the sample rows cyclically
  for (long long r = 0; r < nrows_sample; ++r) {
    roff[r] = lab.size();
    int x = 0;
    while (x < row) {
      lab.push_back((int)(rng() % 1000000));
      start.push_back((unsigned short)x);
      x += 1 + (int)(rng() % 13);
    }
  }
  roff[nrows_sample] = lab.size();
  printf("runs per row %.1f\n", (double)lab.size() / nrows_sample);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] { std::memset((char*)img + nv * 4 / T * t, rep + 1, nv * 4 / T); });
    for (auto& x : th) x.join();
    auto t1 = std::chrono::steady_clock::now();
    th.clear();
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const long long nr = nv / row, r0 = nr * t / T, r1 = nr * (t + 1) / T;
        alignas(64) int buf[1024];
        for (long long r = r0; r < r1; ++r) {
          const long long s = r % nrows_sample;
          const long long a = roff[s], b = roff[s + 1];
          for (long long k = a; k < b; ++k) {
            const int x0 = start[k], x1 = k + 1 < b ? start[k + 1] : (int)row;
            const __m512i v = _mm512_set1_epi32(lab[k]);
            for (int x = x0; x < x1; x += 16) _mm512_storeu_si512(buf + x, v);
          }
          int* dst = img + r * row;  // rows are 4000 B: 16-B aligned
          for (int x = 0; x < row; x += 4) _mm_stream_si128((__m128i*)(dst + x), _mm_load_si128((__m128i*)(buf + x)));
        }
      });
    for (auto& x : th) x.join();
    auto t2 = std::chrono::steady_clock::now();
    printf("threads %d memset %.1f ms (%.1f GB/s)  rle-decode %.1f ms (%.1f GB/s)\n", T,
           std::chrono::duration<double, std::milli>(t1 - t0).count(),
           nv * 4 / 1e6 / std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t2 - t1).count(),
           nv * 4 / 1e6 / std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  return 0;
}
