// C entry points into the reference's own FFT, compiled from
// /root/reference/proj/src/fft.cpp by oracle/Makefile into
// oracle/_ref/libref_fft.so. Test infrastructure: pins oracle.cpp's
// restated radix2() (tests/test_oracle.py, tests/golden/ref_fft.npz).
#include <complex>
#include <cstddef>
#include <stdexcept>

#include "arraymom/fft.hpp"

extern "C" size_t ref_next_pow2(size_t n) { return arraymom::nextPow2(n); }

// Returns 0, or 1 when the reference throws UserError (non power of two).
extern "C" int ref_fft(double* a, size_t n, int inverse) {
  try {
    arraymom::fftInPlace(reinterpret_cast<std::complex<double>*>(a), n, inverse != 0);
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}
