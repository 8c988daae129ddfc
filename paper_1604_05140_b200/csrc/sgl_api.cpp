// C++ mirror of the reference's sgl:: hot-path API on top of the sglgpu C ABI.
// See include/sgl_b200/sgl_transform.hpp.
#include "sgl_b200/sgl_transform.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>

#include "sglgpu.h"

#include <dlfcn.h>

#ifndef SGL_B200_TABLES_DIR
#define SGL_B200_TABLES_DIR ""
#endif

namespace sgl {

namespace {

constexpr double kPi = 3.14159265358979323846;

void check_bandlimit(int B) {
    if (B < 1 || B > 512) {
        throw std::invalid_argument("bandlimit must be in [1, 512], got " + std::to_string(B));
    }
}

// sgl_transform.cpp:18-25
void check_plan_grid(const SampleGrid& grid, const TransformPlan& plan) {
    if (grid.bandlimit != plan.bandlimit) {
        throw std::invalid_argument("transform: grid and plan bandlimits disagree");
    }
    if (grid.values.size() != sample_count(plan.bandlimit)) {
        throw std::invalid_argument("transform: sample grid must have length 8B^3");
    }
}

// sgl_transform.cpp:27-35
void check_plan_coeffs(const SglCoefficients& coeffs, const TransformPlan& plan) {
    if (coeffs.bandlimit != plan.bandlimit) {
        throw std::invalid_argument("transform: coefficient and plan bandlimits disagree");
    }
    if (coeffs.values.size() != coefficient_count(plan.bandlimit)) {
        throw std::invalid_argument("transform: coefficient vector must have length B(B+1)(2B+1)/6");
    }
}

void throw_status(int status) {
    if (status == SGLGPU_OK) return;
    const std::string msg = sglgpu_last_error();
    if (status == SGLGPU_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// CRC-32 (IEEE, reflected 0xEDB88320) -- the zlib crc32 the SGLT store uses
// (precompute_store.cpp:23-28).
std::uint32_t crc32(const unsigned char* p, std::size_t n) {
    static const auto table = [] {
        std::array<std::uint32_t, 256> t{};
        for (std::uint32_t i = 0; i < 256; ++i) {
            std::uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[i] = c;
        }
        return t;
    }();
    std::uint32_t c = 0xFFFFFFFFu;
    for (std::size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

// SGLT reader (precompute_store.hpp:14-30, precompute_store.cpp:59-117).
std::vector<double> read_sglt(const std::filesystem::path& path, std::uint8_t kind, std::uint32_t& B) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open for reading: " + path.string());
    std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    constexpr std::size_t header = 13;
    if (bytes.size() < header + 4) throw std::runtime_error("file too short: " + path.string());
    if (std::memcmp(bytes.data(), "SGLT", 4) != 0) throw std::runtime_error("not a table file: " + path.string());
    std::uint32_t version;
    std::memcpy(&version, bytes.data() + 4, 4);
    if (version != 1) throw std::runtime_error("unsupported format version in " + path.string());
    std::memcpy(&B, bytes.data() + 8, 4);
    if (bytes[12] != kind) throw std::runtime_error("unexpected table kind in " + path.string());
    const std::size_t body = bytes.size() - header - 4;
    if (body % 8 != 0) throw std::runtime_error("payload is not a whole number of doubles: " + path.string());
    std::uint32_t crc;
    std::memcpy(&crc, bytes.data() + bytes.size() - 4, 4);
    if (crc != crc32(bytes.data() + header, body)) throw std::runtime_error("payload checksum mismatch: " + path.string());
    std::vector<double> v(body / 8);
    std::memcpy(v.data(), bytes.data() + header, body);
    return v;
}

// $SGL_TABLES, else the tables/ directory next to this shared library.
std::filesystem::path default_tables_dir() {
    if (const char* env = std::getenv("SGL_TABLES")) return env;
    Dl_info info;
    if (dladdr(reinterpret_cast<void*>(&default_tables_dir), &info) && info.dli_fname) {
        return std::filesystem::path(info.dli_fname).parent_path() / "tables";
    }
    return SGL_B200_TABLES_DIR;
}

// special_functions.cpp:81-88 (kept for API parity; underflows for l+m >~ 172 as in
// the reference -- the GPU path does not use it).
double sph_harm_norm(int l, int m) {
    const double log_ratio = std::lgamma(static_cast<double>(l - m + 1)) - std::lgamma(static_cast<double>(l + m + 1));
    return std::sqrt((2 * l + 1) / (4.0 * kPi) * std::exp(log_ratio));
}

std::mutex g_device_mu;

}  // namespace

std::size_t sample_count(int B) {
    check_bandlimit(B);
    return 8 * static_cast<std::size_t>(B) * B * B;
}

std::size_t coefficient_count(int B) {
    check_bandlimit(B);
    const auto b = static_cast<std::size_t>(B);
    return b * (b + 1) * (2 * b + 1) / 6;
}

int psi_index(int i, int j, int k, int B) {
    check_bandlimit(B);
    if (i < 0 || i >= 2 * B || j < 0 || j >= 2 * B || k < 0 || k >= 2 * B)
        throw std::out_of_range("psi_index: node indices out of range");
    return 4 * B * B * i + 2 * B * j + k;
}

int nu_index(int l, int m) {
    if (l < 0 || m < -l || m > l) throw std::out_of_range("nu_index: require |m| <= l");
    return l * (l + 1) + m;
}

int omega_index(int n, int l, int m) {
    if (n < 1 || l < 0 || l >= n || m < -l || m > l) throw std::out_of_range("omega_index: require |m| <= l < n");
    return static_cast<int>(static_cast<long long>(n - 1) * n * (2 * n - 1) / 6) + l * (l + 1) + m;
}

SphericalRule sphere_rule(int L) {
    if (L < 1) throw std::invalid_argument("sphere_rule: order must be positive");
    SphericalRule rule;
    rule.order = L;
    const int count = 2 * L;
    rule.theta.resize(count);
    rule.phi.resize(count);
    rule.b_raw.resize(count);
    rule.b_cal.resize(count);
    for (int j = 0; j < count; ++j) {
        rule.theta[j] = (2 * j + 1) * kPi / (4.0 * L);
        rule.phi[j] = j * kPi / L;
        double acc = 0.0;
        for (int l = 0; l < L; ++l) acc += std::sin((2 * j + 1) * (2 * l + 1) * kPi / (4.0 * L)) / (2 * l + 1);
        rule.b_raw[j] = std::sin((2 * j + 1) * kPi / (4.0 * L)) * (2.0 / L) * acc;
        rule.b_cal[j] = kPi / L * rule.b_raw[j];
    }
    return rule;
}

RadialRule load_radial_rule(const std::filesystem::path& path) {
    std::uint32_t B = 0;
    const auto v = read_sglt(path, 1, B);
    if (v.size() != 6 * static_cast<std::size_t>(B))
        throw std::runtime_error("payload length does not match the declared bandlimit: " + path.string());
    RadialRule r;
    r.order = 2 * static_cast<int>(B);
    r.r.assign(v.begin(), v.begin() + 2 * B);
    r.a.assign(v.begin() + 2 * B, v.begin() + 4 * B);
    r.a_mod.assign(v.begin() + 4 * B, v.end());
    return r;
}

SphericalRule load_spherical_rule(const std::filesystem::path& path) {
    std::uint32_t B = 0;
    const auto v = read_sglt(path, 2, B);
    if (v.size() != 8 * static_cast<std::size_t>(B))
        throw std::runtime_error("payload length does not match the declared bandlimit: " + path.string());
    SphericalRule s;
    s.order = static_cast<int>(B);
    const std::size_t n = 2 * B;
    s.theta.assign(v.begin(), v.begin() + n);
    s.phi.assign(v.begin() + n, v.begin() + 2 * n);
    s.b_raw.assign(v.begin() + 2 * n, v.begin() + 3 * n);
    s.b_cal.assign(v.begin() + 3 * n, v.end());
    return s;
}

// sgl_transform.cpp:52-88 (validation and the derived per-node / per-order vectors)
TransformPlan TransformPlan::assemble(int B, RadialRule radial, SphericalRule sphere) {
    if (B < 1) throw std::invalid_argument("TransformPlan: bandlimit must be positive");
    if (radial.order != 2 * B) throw std::invalid_argument("TransformPlan: radial rule order must be 2B");
    if (sphere.order != B) throw std::invalid_argument("TransformPlan: spherical tables must have order B");
    TransformPlan plan;
    plan.bandlimit = B;
    plan.radial = std::move(radial);
    plan.sphere.order = B;
    plan.sphere.rule = std::move(sphere);
    plan.exp_neg_r2.resize(plan.radial.r.size());
    for (std::size_t i = 0; i < plan.radial.r.size(); ++i)
        plan.exp_neg_r2[i] = std::exp(-plan.radial.r[i] * plan.radial.r[i]);
    plan.cos_theta.resize(plan.sphere.rule.theta.size());
    for (std::size_t j = 0; j < plan.cos_theta.size(); ++j) plan.cos_theta[j] = std::cos(plan.sphere.rule.theta[j]);
    plan.seed_norm.resize(B);
    for (int l = 0; l < B; ++l) plan.seed_norm[l] = std::sqrt(2.0 * std::exp(-std::lgamma(l + 1.5)));
    plan.m_norm.resize(static_cast<std::size_t>(B) * B);
    for (int l = 0; l < B; ++l) {
        for (int m = -l; m <= l; ++m) {
            const int am = std::abs(m);
            const double sign = (m < 0 && am % 2 != 0) ? -1.0 : 1.0;
            plan.m_norm[static_cast<std::size_t>(nu_index(l, m))] = sign * sph_harm_norm(l, am);
        }
    }
    return plan;
}

TransformPlan TransformPlan::compute(int B) {
    if (B < 1) throw std::invalid_argument("TransformPlan: bandlimit must be positive");
    const auto dir = default_tables_dir();
    const auto path = dir / ("radial_rule_B" + std::to_string(B) + ".sglt");
    if (!std::filesystem::exists(path)) {
        throw QuadratureError("half_range_hermite_rule: no tabulated rule of order " + std::to_string(2 * B) +
                              " in " + dir.string() +
                              " (generate it with python -m paper_1604_05140_b200.tables.gen_radial_rules " +
                              std::to_string(B) + ")");
    }
    return assemble(B, load_radial_rule(path), sphere_rule(B));
}

TransformPlan TransformPlan::from_tables(const std::filesystem::path& dir, int B) {
    auto radial = load_radial_rule(dir / ("radial_rule_B" + std::to_string(B) + ".sglt"));
    const auto sp = dir / ("sphere_rule_B" + std::to_string(B) + ".sglt");
    auto sphere = std::filesystem::exists(sp) ? load_spherical_rule(sp) : sphere_rule(B);
    return assemble(B, std::move(radial), std::move(sphere));
}

sglgpu_plan* TransformPlan::device_plan() const {
    std::lock_guard<std::mutex> lock(g_device_mu);
    auto& slot = const_cast<std::shared_ptr<sglgpu_plan>&>(device);
    if (!slot) {
        sglgpu_plan_desc d{};
        d.bandlimit = bandlimit;
        d.r = radial.r.data();
        d.a_mod = radial.a_mod.data();
        d.b_cal = sphere.rule.b_cal.data();
        d.device = -1;
        sglgpu_plan* p = nullptr;
        throw_status(sglgpu_plan_create(&d, &p));
        slot = std::shared_ptr<sglgpu_plan>(p, [](sglgpu_plan* q) { sglgpu_plan_destroy(q); });
    }
    return slot.get();
}

SglCoefficients fsglft(const SampleGrid& grid, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_grid(grid, plan);
    SglCoefficients out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(coefficient_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_forward(plan.device_plan(), reinterpret_cast<const double*>(grid.values.data()),
                                reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SampleGrid ifsglft(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_coeffs(coeffs, plan);
    SampleGrid out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(sample_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_inverse(plan.device_plan(), reinterpret_cast<const double*>(coeffs.values.data()),
                                reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SglCoefficients dsglft_separated(const SampleGrid& grid, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_grid(grid, plan);
    SglCoefficients out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(coefficient_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_forward_separated(plan.device_plan(), reinterpret_cast<const double*>(grid.values.data()),
                                          reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST, nullptr));
    return out;
}

SampleGrid idsglft_separated(const SglCoefficients& coeffs, const TransformPlan& plan, unsigned /*threads*/) {
    check_plan_coeffs(coeffs, plan);
    SampleGrid out;
    out.bandlimit = plan.bandlimit;
    out.values.assign(sample_count(plan.bandlimit), cplx(0.0));
    throw_status(sglgpu_inverse_separated(plan.device_plan(), reinterpret_cast<const double*>(coeffs.values.data()),
                                          reinterpret_cast<double*>(out.values.data()), 1, SGLGPU_MEM_HOST,
                                          nullptr));
    return out;
}

void fsglft_batch(const TransformPlan& plan, const cplx* samples, cplx* coeffs, std::size_t batch,
                  bool device_pointers, void* stream) {
    throw_status(sglgpu_forward(plan.device_plan(), reinterpret_cast<const double*>(samples),
                                reinterpret_cast<double*>(coeffs), batch,
                                device_pointers ? SGLGPU_MEM_DEVICE : SGLGPU_MEM_HOST, stream));
}

void ifsglft_batch(const TransformPlan& plan, const cplx* coeffs, cplx* samples, std::size_t batch,
                   bool device_pointers, void* stream) {
    throw_status(sglgpu_inverse(plan.device_plan(), reinterpret_cast<const double*>(coeffs),
                                reinterpret_cast<double*>(samples), batch,
                                device_pointers ? SGLGPU_MEM_DEVICE : SGLGPU_MEM_HOST, stream));
}

// sgl_transform.cpp:350-366
RoundtripError roundtrip_error(std::span<const cplx> reference, std::span<const cplx> actual) {
    if (reference.size() != actual.size()) throw std::invalid_argument("roundtrip_error: vector lengths disagree");
    RoundtripError err;
    for (std::size_t i = 0; i < reference.size(); ++i) {
        if (!std::isfinite(actual[i].real()) || !std::isfinite(actual[i].imag())) ++err.nonfinite;
        const double diff = std::abs(reference[i] - actual[i]);
        err.max_abs = std::max(err.max_abs, diff);
        const double mag = std::abs(reference[i]);
        if (mag == 0.0) {
            ++err.skipped_zero;
        } else {
            err.max_rel = std::max(err.max_rel, diff / mag);
        }
    }
    return err;
}

}  // namespace sgl
