// Operator / vector files of the reference: "BTOP" and
// "BTVC", 64-byte little-endian headers (proj/include/btoep/io.hpp:12-18,
// src/io.cpp:13-240). Files are streamed, never loaded whole, so an operator
// larger than host memory goes straight into HBM:
//   btg_load_operator  time-domain file  -> sensor-row slabs -> btg_setup_rows
//                      frequency-domain  -> the N_t+1 stored blocks -> F-hat
//   btg_save_operator  F-hat -> frequency-domain file in the reference's full
//                      2 N_t layout (upper half by conjugate symmetry), one
//                      block at a time.
// Byte-exact with the reference's writer for the same values.
#include <cuda_runtime.h>

#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/btg.h"

// shared with btg_capi.cu (defined there, C linkage, not declared in btg.h)
extern "C" {
btg_status btg_internal_fail(btg_status s, const char* msg);
btg_status btg_internal_upload_spectrum_block(btg_op op, size_t f, const double* block_c128);
btg_status btg_internal_mark_ready(btg_op op);
}

namespace {

constexpr size_t kHeader = 64;
constexpr uint32_t kVersion = 1;

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

btg_status ferr(const std::string& m) { return btg_internal_fail(BTG_EFORMAT, m.c_str()); }

void put_u32(unsigned char* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}
void put_u64(unsigned char* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}
uint32_t get_u32(const unsigned char* p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[i]) << (8 * i);
    return v;
}
uint64_t get_u64(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    return v;
}

bool read_at(FILE* f, uint64_t off, void* dst, size_t n) {
    if (std::fseek(f, static_cast<long>(off), SEEK_SET) != 0) return false;
    return std::fread(dst, 1, n, f) == n;
}

uint64_t file_size(FILE* f) {
    std::fseek(f, 0, SEEK_END);
    const long s = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    return s < 0 ? 0 : static_cast<uint64_t>(s);
}

}  // namespace

extern "C" {

btg_status btg_peek_operator(const char* path, btg_file_header* out) {
    if (!path || !out) return btg_internal_fail(BTG_EARG, "null argument");
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) return ferr(std::string("cannot open '") + path + "'");
    unsigned char h[kHeader];
    if (!read_at(fh.f, 0, h, kHeader)) return ferr(std::string("'") + path + "' is too short for an operator header");
    if (std::memcmp(h, "BTOP", 4) != 0) return ferr(std::string("'") + path + "' is not an operator file (bad magic)");
    if (get_u32(h + 4) != kVersion) return ferr(std::string("'") + path + "': unsupported operator format version");
    const uint32_t ordering = get_u32(h + 8), domain = get_u32(h + 12), scalar = get_u32(h + 40);
    if (ordering > 1) return ferr(std::string("'") + path + "': bad ordering flag");
    if (domain > 1) return ferr(std::string("'") + path + "': bad domain flag");
    if (scalar > 1) return ferr(std::string("'") + path + "': bad scalar kind");
    out->ordering = (int)ordering;
    out->domain = (int)domain;
    out->num_sensors = get_u64(h + 16);
    out->num_sources = get_u64(h + 24);
    out->num_steps = get_u64(h + 32);
    out->complex_scalar = (int)scalar;
    const uint64_t per = domain == 0 ? 8 : 16;
    const uint64_t nblk = domain == 0 ? out->num_steps : 2 * out->num_steps;
    const uint64_t want = kHeader + per * nblk * out->num_sensors * out->num_sources;
    if (file_size(fh.f) != want)
        return ferr(std::string("'") + path + "': payload size does not match the header");
    return BTG_OK;
}

btg_status btg_load_operator(const char* path, int precision, int device, btg_op* out) {
    btg_file_header h{};
    btg_status s = btg_peek_operator(path, &h);
    if (s != BTG_OK) return s;
    return btg_load_operator_rect(path, 0, h.num_sensors, 0, h.num_sources, precision, device, out);
}

btg_status btg_load_operator_rect(const char* path, size_t i0, size_t i1, size_t j0, size_t j1, int precision,
                                  int device, btg_op* out) {
    if (!out) return btg_internal_fail(BTG_EARG, "null output handle");
    *out = nullptr;
    btg_file_header h{};
    btg_status s = btg_peek_operator(path, &h);
    if (s != BTG_OK) return s;
    if (h.ordering != 0) return ferr(std::string("'") + path + "': operators must be TOSI-ordered");
    if ((h.domain == 0) == (h.complex_scalar != 0))
        return ferr(std::string("'") + path + "': domain and scalar kind disagree");
    const size_t ND = h.num_sensors, NM = h.num_sources, nt = h.num_steps;
    if (i0 >= i1 || i1 > ND || j0 >= j1 || j1 > NM)
        return btg_internal_fail(BTG_EDIM, "load_operator_rect: rectangle outside the operator");
    const size_t nd = i1 - i0, nm = j1 - j0;
    btg_op op = nullptr;
    s = btg_create(nd, nm, nt, precision, device, &op);
    if (s != BTG_OK) return s;
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) {
        btg_destroy(op);
        return ferr(std::string("cannot open '") + path + "'");
    }
    auto bail = [&](btg_status st) {
        btg_destroy(op);
        return st;
    };
    // Rows of the rectangle are contiguous (nm values) in every stored block.
    if (h.domain == 0) {
        // time domain: sensor-row slabs (N_t, rows, nm) through btg_setup_rows
        // (the reference's partition_operator(CompactP2O), distributed.cpp:179-196)
        const size_t row_bytes = nt * nm * sizeof(double);
        const size_t rows = std::max<size_t>(1, std::min<size_t>(nd, (size_t(1) << 30) / row_bytes));
        std::vector<double> slab(rows * nt * nm);
        for (size_t r0 = 0; r0 < nd; r0 += rows) {
            const size_t r = std::min(rows, nd - r0);
            for (size_t k = 0; k < nt; ++k)
                for (size_t i = 0; i < r; ++i) {
                    const uint64_t off = kHeader + (((uint64_t)k * ND + i0 + r0 + i) * NM + j0) * sizeof(double);
                    if (!read_at(fh.f, off, slab.data() + (k * r + i) * nm, nm * sizeof(double)))
                        return bail(ferr(std::string("'") + path + "': file truncated"));
                }
            s = btg_setup_rows(op, slab.data(), r0, r0 + r, 0u);
            if (s != BTG_OK) return bail(s);
        }
    } else {
        // frequency domain: blocks f = 0..N_t of the stored 2 N_t, rectangle only
        // (partition_operator(SpectralP2O), distributed.cpp:198-218: no re-setup)
        std::vector<double> blk(2 * nd * nm);
        for (size_t f = 0; f <= nt; ++f) {
            for (size_t i = 0; i < nd; ++i) {
                const uint64_t off = kHeader + (((uint64_t)f * ND + i0 + i) * NM + j0) * 16;
                if (!read_at(fh.f, off, blk.data() + 2 * i * nm, nm * 16))
                    return bail(ferr(std::string("'") + path + "': file truncated"));
            }
            s = btg_internal_upload_spectrum_block(op, f, blk.data());
            if (s != BTG_OK) return bail(s);
        }
        s = btg_internal_mark_ready(op);
        if (s != BTG_OK) return bail(s);
    }
    *out = op;
    return BTG_OK;
}

btg_status btg_save_operator(btg_op op, const char* path) {
    if (!op || !path) return btg_internal_fail(BTG_EARG, "null argument");
    size_t nd = 0, nm = 0, nt = 0;
    int prec = 0;
    btg_status s = btg_get_dims(op, &nd, &nm, &nt, &prec);
    if (s != BTG_OK) return s;
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) return ferr(std::string("cannot open '") + path + "' for writing");
    unsigned char h[kHeader] = {};
    std::memcpy(h, "BTOP", 4);
    put_u32(h + 4, kVersion);
    put_u32(h + 8, 0);   // TOSI
    put_u32(h + 12, 1);  // frequency domain
    put_u64(h + 16, nd);
    put_u64(h + 24, nm);
    put_u64(h + 32, nt);
    put_u32(h + 40, 1);  // complex
    if (std::fwrite(h, 1, kHeader, fh.f) != kHeader) return ferr("failed writing the header");
    // stored half, block by block, then the conjugate-symmetric upper half
    std::vector<std::complex<double>> blk(nd * nm);
    for (size_t f = 0; f < 2 * nt; ++f) {
        const size_t src = f <= nt ? f : 2 * nt - f;
        s = btg_export_spectrum_block(op, src, reinterpret_cast<double*>(blk.data()));
        if (s != BTG_OK) return s;
        if (f > nt)
            for (auto& v : blk) v = std::conj(v);
        if (std::fwrite(blk.data(), sizeof(std::complex<double>), blk.size(), fh.f) != blk.size())
            return ferr("failed writing the payload");
    }
    return BTG_OK;
}

// io::write_operator(CompactP2O) (io.cpp:97-111): time-domain TOSI file.
btg_status btg_write_compact(const char* path, const double* blocks, size_t nd, size_t nm, size_t nt) {
    if (!path || !blocks) return btg_internal_fail(BTG_EARG, "null argument");
    if (nd == 0 || nm == 0 || nt == 0)
        return btg_internal_fail(BTG_EDIM, "compact operator: all dimensions must be positive");
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) return ferr(std::string("cannot open '") + path + "' for writing");
    unsigned char h[kHeader] = {};
    std::memcpy(h, "BTOP", 4);
    put_u32(h + 4, kVersion);
    put_u32(h + 8, 0);   // TOSI
    put_u32(h + 12, 0);  // time domain
    put_u64(h + 16, nd);
    put_u64(h + 24, nm);
    put_u64(h + 32, nt);
    put_u32(h + 40, 0);  // real
    if (std::fwrite(h, 1, kHeader, fh.f) != kHeader) return ferr("failed writing the header");
    const size_t n = nt * nd * nm;
    if (std::fwrite(blocks, sizeof(double), n, fh.f) != n) return ferr("failed writing the payload");
    return BTG_OK;
}

// io::read_compact_operator (io.cpp:159-180); blocks == NULL queries the dimensions.
btg_status btg_read_compact(const char* path, double* blocks, size_t capacity, size_t* nd, size_t* nm,
                            size_t* nt) {
    btg_file_header h{};
    btg_status s = btg_peek_operator(path, &h);
    if (s != BTG_OK) return s;
    if (h.domain != 0 || h.complex_scalar)
        return ferr(std::string("'") + path +
                    "' holds a frequency-domain operator; a time-domain compact operator was expected");
    if (h.ordering != 0) return ferr(std::string("'") + path + "': compact operators must be TOSI-ordered");
    if (nd) *nd = h.num_sensors;
    if (nm) *nm = h.num_sources;
    if (nt) *nt = h.num_steps;
    if (!blocks) return BTG_OK;
    const size_t n = h.num_steps * h.num_sensors * h.num_sources;
    if (capacity < n) return btg_internal_fail(BTG_EDIM, "read_compact: destination too small");
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f || !read_at(fh.f, kHeader, blocks, n * sizeof(double))) return ferr("file truncated");
    return BTG_OK;
}

btg_status btg_write_vector(const char* path, const double* values, size_t spatial_dim, size_t num_steps,
                            int ordering) {
    if (!path || (!values && spatial_dim * num_steps != 0)) return btg_internal_fail(BTG_EARG, "null argument");
    if (ordering != 0 && ordering != 1) return btg_internal_fail(BTG_EORDER, "ordering must be 0 (TOSI) or 1 (SOTI)");
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) return ferr(std::string("cannot open '") + path + "' for writing");
    unsigned char h[kHeader] = {};
    std::memcpy(h, "BTVC", 4);
    put_u32(h + 4, (uint32_t)ordering);
    put_u64(h + 8, spatial_dim);
    put_u64(h + 16, num_steps);
    if (std::fwrite(h, 1, kHeader, fh.f) != kHeader) return ferr("failed writing the header");
    const size_t n = spatial_dim * num_steps;
    if (std::fwrite(values, sizeof(double), n, fh.f) != n) return ferr("failed writing the payload");
    return BTG_OK;
}

btg_status btg_read_vector(const char* path, double* values, size_t capacity, size_t* spatial_dim,
                           size_t* num_steps, int* ordering) {
    if (!path) return btg_internal_fail(BTG_EARG, "null argument");
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) return ferr(std::string("cannot open '") + path + "'");
    unsigned char h[kHeader];
    if (!read_at(fh.f, 0, h, kHeader)) return ferr(std::string("'") + path + "' is too short for a vector header");
    if (std::memcmp(h, "BTVC", 4) != 0) return ferr(std::string("'") + path + "' is not a vector file (bad magic)");
    const uint32_t ord = get_u32(h + 4);
    if (ord > 1) return ferr(std::string("'") + path + "': bad ordering flag");
    const uint64_t sp = get_u64(h + 8), st = get_u64(h + 16);
    if (file_size(fh.f) != kHeader + sp * st * 8)
        return ferr(std::string("'") + path + "': payload size does not match the header");
    if (spatial_dim) *spatial_dim = sp;
    if (num_steps) *num_steps = st;
    if (ordering) *ordering = (int)ord;
    if (!values) return BTG_OK;  // size query
    if (capacity < sp * st) return btg_internal_fail(BTG_EDIM, "read_vector: destination too small");
    if (!read_at(fh.f, kHeader, values, sp * st * 8)) return ferr("file truncated");
    return BTG_OK;
}

}  // extern "C"
