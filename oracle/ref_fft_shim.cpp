// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Stand-in for the reference's FFTW wrapper (/root/reference/proj/src/fft.cpp),
// which needs FFTW3 (absent from this image). It implements exactly the two
// functions declared at /root/reference/proj/include/btoep/fft.hpp:10,13:
//
//   forward(data, n, count)  unnormalized DFT, sign -1   (fft.cpp:38-40)
//   inverse(data, n, count)  DFT with sign +1, then x 1/n (fft.cpp:42-46)
//
// in place over `count` contiguous length-n transforms. The algorithm is a
// mixed-radix Stockham autosort (radix 4/2/3/5 butterflies, a generic odd
// radix for small primes) with Bluestein's chirp-z convolution for prime
// factors > 61, so every length is O(n log n). Plans (twiddle tables and
// factorizations) are cached per (n, sign) behind a mutex, mirroring the
// reference's planner serialization (fft.cpp:12-33).
#include <cmath>
#include <complex>
#include <cstddef>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace btoep::fft {
namespace {

using cd = std::complex<double>;

// exp(sign * 2*pi*i * num / den), argument reduced exactly in integers first.
cd unit_root(long long num, long long den, int sign) {
    num %= den;
    if (num < 0) num += den;
    const long double ang = 2.0L * 3.14159265358979323846264338327950288L *
                            static_cast<long double>(num) / static_cast<long double>(den);
    return {static_cast<double>(std::cos(ang)), static_cast<double>(sign * std::sin(ang))};
}

struct Plan;
std::shared_ptr<const Plan> get_plan(std::size_t n, int sign);

struct Plan {
    std::size_t n = 0;
    int sign = -1;
    std::vector<std::size_t> factors;  // Stockham radices (product n) unless bluestein
    std::vector<cd> tw;                // tw[k] = exp(sign*2*pi*i*k/n)
    // Bluestein
    bool bluestein = false;
    std::size_t m = 0;             // power-of-two convolution length
    std::vector<cd> chirp;         // exp(sign*pi*i*k^2/n), k < n
    std::vector<cd> kernel_hat;    // FFT_m of conj chirp (wrapped)
    std::shared_ptr<const Plan> sub_fwd, sub_inv;
};

std::vector<std::size_t> factorize(std::size_t n, bool& needs_bluestein) {
    std::vector<std::size_t> f;
    needs_bluestein = false;
    while (n % 4 == 0) { f.push_back(4); n /= 4; }
    while (n % 2 == 0) { f.push_back(2); n /= 2; }
    for (std::size_t p = 3; p * p <= n; p += 2)
        while (n % p == 0) {
            if (p > 61) needs_bluestein = true;
            f.push_back(p);
            n /= p;
        }
    if (n > 1) {
        if (n > 61) needs_bluestein = true;
        f.push_back(n);
    }
    return f;
}

void stockham(const Plan& p, cd* x, cd* work) {
    const std::size_t n = p.n;
    cd* src = x;
    cd* dst = work;
    std::size_t ns = 1;
    cd v[64];
    cd out[64];
    for (std::size_t r : p.factors) {
        const std::size_t stride = n / r;
        const std::size_t tw_step = n / (ns * r);
        for (std::size_t j = 0; j < stride; ++j) {
            const std::size_t k = j % ns;
            for (std::size_t q = 0; q < r; ++q) {
                cd a = src[j + q * stride];
                if (q && k) a *= p.tw[(k * q * tw_step) % n];
                v[q] = a;
            }
            // r-point DFT with root exp(sign*2*pi*i/r) = tw[n/r]
            if (r == 2) {
                out[0] = v[0] + v[1];
                out[1] = v[0] - v[1];
            } else if (r == 4) {
                const cd a0 = v[0] + v[2], a1 = v[0] - v[2];
                const cd b0 = v[1] + v[3], b1 = v[1] - v[3];
                const cd jb1 = p.sign < 0 ? cd(b1.imag(), -b1.real()) : cd(-b1.imag(), b1.real());
                out[0] = a0 + b0;
                out[1] = a1 + jb1;
                out[2] = a0 - b0;
                out[3] = a1 - jb1;
            } else {
                for (std::size_t q = 0; q < r; ++q) {
                    cd acc = v[0];
                    for (std::size_t s = 1; s < r; ++s) acc += v[s] * p.tw[((q * s) % r) * stride];
                    out[q] = acc;
                }
            }
            const std::size_t base = (j / ns) * ns * r + k;
            for (std::size_t q = 0; q < r; ++q) dst[base + q * ns] = out[q];
        }
        std::swap(src, dst);
        ns *= r;
    }
    if (src != x)
        for (std::size_t i = 0; i < n; ++i) x[i] = src[i];
}

void execute(const Plan& p, cd* x, std::vector<cd>& scratch);

void bluestein(const Plan& p, cd* x, std::vector<cd>& scratch) {
    const std::size_t n = p.n, m = p.m;
    std::vector<cd> a(m, cd(0.0, 0.0));
    for (std::size_t k = 0; k < n; ++k) a[k] = x[k] * p.chirp[k];
    std::vector<cd> inner;
    execute(*p.sub_fwd, a.data(), inner);
    for (std::size_t k = 0; k < m; ++k) a[k] *= p.kernel_hat[k];
    execute(*p.sub_inv, a.data(), inner);
    const double inv_m = 1.0 / static_cast<double>(m);
    for (std::size_t k = 0; k < n; ++k) x[k] = a[k] * inv_m * p.chirp[k];
    (void)scratch;
}

void execute(const Plan& p, cd* x, std::vector<cd>& scratch) {
    if (p.n <= 1) return;
    if (p.bluestein) {
        bluestein(p, x, scratch);
        return;
    }
    if (scratch.size() < p.n) scratch.resize(p.n);
    stockham(p, x, scratch.data());
}

std::shared_ptr<const Plan> build_plan(std::size_t n, int sign) {
    auto p = std::make_shared<Plan>();
    p->n = n;
    p->sign = sign;
    bool blue = false;
    p->factors = factorize(n, blue);
    if (!blue) {
        p->tw.resize(n);
        for (std::size_t k = 0; k < n; ++k) p->tw[k] = unit_root(static_cast<long long>(k),
                                                                  static_cast<long long>(n), sign);
        return p;
    }
    p->bluestein = true;
    std::size_t m = 1;
    while (m < 2 * n - 1) m *= 2;
    p->m = m;
    p->chirp.resize(n);
    const long long two_n = 2 * static_cast<long long>(n);
    for (std::size_t k = 0; k < n; ++k) {
        const long long kk = static_cast<long long>(k);
        p->chirp[k] = unit_root((kk * kk) % two_n, two_n, sign);  // exp(sign*pi*i*k^2/n)
    }
    p->sub_fwd = get_plan(m, -1);
    p->sub_inv = get_plan(m, +1);
    std::vector<cd> b(m, cd(0.0, 0.0));
    for (std::size_t k = 0; k < n; ++k) {
        b[k] = std::conj(p->chirp[k]);
        if (k) b[m - k] = std::conj(p->chirp[k]);
    }
    std::vector<cd> inner;
    execute(*p->sub_fwd, b.data(), inner);
    p->kernel_hat = std::move(b);
    return p;
}

std::mutex& planner_mutex() {
    static std::mutex mtx;
    return mtx;
}

std::shared_ptr<const Plan> get_plan(std::size_t n, int sign) {
    static std::map<std::pair<std::size_t, int>, std::shared_ptr<const Plan>> cache;
    {
        std::lock_guard<std::mutex> lock(planner_mutex());
        auto it = cache.find({n, sign});
        if (it != cache.end()) return it->second;
    }
    auto plan = build_plan(n, sign);  // may recurse into get_plan (Bluestein)
    std::lock_guard<std::mutex> lock(planner_mutex());
    auto [it, inserted] = cache.emplace(std::make_pair(n, sign), plan);
    return it->second;
}

void transform(cd* data, std::size_t n, std::size_t count, int sign) {
    if (n == 0 || count == 0) return;
    auto plan = get_plan(n, sign);
    std::vector<cd> scratch;
    for (std::size_t b = 0; b < count; ++b) execute(*plan, data + b * n, scratch);
}

}  // namespace

void forward(std::complex<double>* data, std::size_t n, std::size_t count) {
    transform(data, n, count, -1);
}

void inverse(std::complex<double>* data, std::size_t n, std::size_t count) {
    transform(data, n, count, +1);
    const double scale = 1.0 / static_cast<double>(n);
    for (std::size_t i = 0; i < n * count; ++i) data[i] *= scale;
}

}  // namespace btoep::fft
