// Host half of the run-coded label transport (labelrun.cu): expand x-rows of
// runs into the caller's int32 image.  Compiled by g++ -O3; the AVX-512 fill
// is chosen at run time (__builtin_cpu_supports), SSE2 otherwise.
#include <immintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace vxb {

namespace {

// One row: runs [L, X) of n runs -> b[0, n0) (b has n0 + 16 ints of slack).
__attribute__((target("avx512f"))) void fill_row_avx512(const int* L, const unsigned short* X, int n, int n0,
                                                        int* b) {
  for (int k = 0; k < n; ++k) {
    const int a = std::min<int>(X[k], n0);
    const int e = k + 1 < n ? std::min<int>(X[k + 1], n0) : n0;
    const __m512i v = _mm512_set1_epi32(L[k]);
    for (int x = a; x < e; x += 16) _mm512_storeu_si512(reinterpret_cast<void*>(b + x), v);
  }
}

// b -> out (out 16-byte aligned, n0 % 4 == 0): 16-byte streaming stores up
// to the first 64-byte boundary, whole-line streaming stores, then the tail.
__attribute__((target("avx512f"))) void stream_row_avx512(int32_t* out, const int* b, int n0) {
  int x = 0;
  for (; x < n0 && (reinterpret_cast<uintptr_t>(out + x) & 63) != 0; x += 4)
    _mm_stream_si128(reinterpret_cast<__m128i*>(out + x), _mm_loadu_si128(reinterpret_cast<const __m128i*>(b + x)));
  for (; x + 16 <= n0; x += 16)
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + x), _mm512_loadu_si512(reinterpret_cast<const void*>(b + x)));
  for (; x < n0; x += 4)
    _mm_stream_si128(reinterpret_cast<__m128i*>(out + x), _mm_loadu_si128(reinterpret_cast<const __m128i*>(b + x)));
}

// The packed form: run k is L[k] = label << xbits | first x.
__attribute__((target("avx512f"))) void fill_row_packed_avx512(const unsigned* L, int n, int n0, int xbits, int* b) {
  const unsigned mask = (1u << xbits) - 1u;
  int a = 0;
  for (int k = 0; k < n; ++k) {
    const unsigned u = L[k];
    const int e = k + 1 < n ? std::min<int>((int)(L[k + 1] & mask), n0) : n0;
    const __m512i v = _mm512_set1_epi32((int)(u >> xbits));
    for (int x = a; x < e; x += 16) _mm512_storeu_si512(reinterpret_cast<void*>(b + x), v);
    a = e;
  }
}

void fill_row_packed_sse2(const unsigned* L, int n, int n0, int xbits, int* b) {
  const unsigned mask = (1u << xbits) - 1u;
  int a = 0;
  for (int k = 0; k < n; ++k) {
    const unsigned u = L[k];
    const int e = k + 1 < n ? std::min<int>((int)(L[k + 1] & mask), n0) : n0;
    const __m128i v = _mm_set1_epi32((int)(u >> xbits));
    for (int x = a; x < e; x += 4) _mm_storeu_si128(reinterpret_cast<__m128i*>(b + x), v);
    a = e;
  }
}

void fill_row_sse2(const int* L, const unsigned short* X, int n, int n0, int* b) {
  for (int k = 0; k < n; ++k) {
    const int a = std::min<int>(X[k], n0);
    const int e = k + 1 < n ? std::min<int>(X[k + 1], n0) : n0;
    const __m128i v = _mm_set1_epi32(L[k]);
    for (int x = a; x < e; x += 4) _mm_storeu_si128(reinterpret_cast<__m128i*>(b + x), v);
  }
}

}  // namespace

// Rows [r0, r1) of a run-coded chunk: rows[2 r] = offset of row r's runs,
// rows[2 r + 1] = their count; row r goes to dst + r n0.
void run_decode_rows(const int* rows, const int* rlab, const unsigned short* rx, long long r0, long long r1,
                     int n0, int xbits, int32_t* dst, std::vector<int>& buf) {
  if ((long long)buf.size() < n0 + 32) buf.assign(n0 + 32, 0);
  int* b = buf.data() + ((16 - (reinterpret_cast<uintptr_t>(buf.data()) & 15) / 4) & 3);  // 16-byte aligned
  static const bool avx512 = __builtin_cpu_supports("avx512f");
  const bool stream = (n0 % 4) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  for (long long r = r0; r < r1; ++r) {
    const int off = rows[2 * r], n = rows[2 * r + 1];
    if (xbits > 0 && avx512)
      fill_row_packed_avx512(reinterpret_cast<const unsigned*>(rlab) + off, n, n0, xbits, b);
    else if (xbits > 0)
      fill_row_packed_sse2(reinterpret_cast<const unsigned*>(rlab) + off, n, n0, xbits, b);
    else if (avx512)
      fill_row_avx512(rlab + off, rx + off, n, n0, b);
    else
      fill_row_sse2(rlab + off, rx + off, n, n0, b);
    int32_t* out = dst + r * (long long)n0;
    if (stream && avx512) {
      stream_row_avx512(out, b, n0);
    } else if (stream) {
      for (int x = 0; x < n0; x += 4)
        _mm_stream_si128(reinterpret_cast<__m128i*>(out + x), _mm_load_si128(reinterpret_cast<const __m128i*>(b + x)));
    } else {
      std::memcpy(out, b, sizeof(int32_t) * (size_t)n0);
    }
  }
  if (stream) _mm_sfence();
}

}  // namespace vxb
