// Host-side probe: expand nelt packed lower triangles (m(m+1)/2 doubles each)
// into full column-major m x m slices on T threads; prints GB/s of bytes
// written. g++ -O3 -march=native -pthread host_unpack.cpp -o host_unpack
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  const int m = 40, nelt = argc > 1 ? atoi(argv[1]) : 196608;
  const int ns = m * (m + 1) / 2;
  std::vector<double> packed(size_t(nelt) * ns, 1.0);
  double* out = static_cast<double*>(aligned_alloc(64, size_t(nelt) * m * m * 8));
  for (size_t i = 0; i < size_t(nelt) * m * m; i += 512) out[i] = 0.0;  // touch pages
  for (int T : {1, 4, 8, 16, 32}) {
    auto run = [&] {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          for (long K = long(nelt) * t / T; K < long(nelt) * (t + 1) / T; ++K) {
            const double* p = packed.data() + K * ns;
            double* o = out + K * m * m;
            for (int c = 0; c < m; ++c) {  // column c of the lower triangle: rows c..m-1
              const double* pc = p + c * m - c * (c - 1) / 2 - c;  // start of column c (row index r at pc[r])
              for (int r = c; r < m; ++r) {
                const double v = pc[r];
                o[r + c * m] = v;
                o[c + r * m] = v;
              }
            }
          }
        });
      for (auto& x : th) x.join();
    };
    run();
    const auto t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < 3; ++rep) run();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 3;
    printf("threads %d: %.1f ms, %.1f GB/s written\n", T, s * 1e3, double(nelt) * m * m * 8 / s / 1e9);
  }
  return 0;
}
