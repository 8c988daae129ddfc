// Host side of the C++ mirror that is not a transform: the layouts
// (indexing.cpp), the quadrature helpers (quadrature.cpp:189-242), the SGLT
// table files (precompute_store.cpp), the Legendre DCT table of the plan
// (spherical_transform.cpp:31-86) and the scalar closed forms of the basis
// (special_functions.cpp) -- the reference's public API around fsglft /
// ifsglft.  Headers: include/sgl/*.hpp.  The special functions and the DCT
// table use fully normalized recurrences in long double (finite at every
// bandlimit); the reference's unnormalized seeds under/overflow for
// l + |m| >~ 172, where the two differ.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include "sgl/indexing.hpp"
#include "sgl/precompute_store.hpp"
#include "sgl/quadrature.hpp"
#include "sgl/special_functions.hpp"
#include "sgl/spherical_transform.hpp"

#include <dlfcn.h>

namespace sgl {

namespace {

constexpr long double kPiL = 3.141592653589793238462643383279502884L;

void check_bandlimit(int B) {
    if (B < 1 || B > 512) throw std::invalid_argument("bandlimit must be in [1, 512], got " + std::to_string(B));
}

long long degree_offset(long long n) { return (n - 1) * n * (2 * n - 1) / 6; }

int isqrt(int v) {
    int s = static_cast<int>(std::sqrt(static_cast<double>(v)));
    while (s > 0 && s * s > v) --s;
    while ((s + 1) * (s + 1) <= v) ++s;
    return s;
}

// Fully normalized Pbar_{l,m}(t) = M_lm P_lm(t) for l = m .. L-1 (Condon-Shortley
// phase included): Pbar_mm from a log-space product, then the normalized
// three-term recurrence.  out[l - m].
void pbar_column(int m, int L, long double t, long double* out) {
    const long double s2 = (1.0L - t) * (1.0L + t);
    long double lg = 0.5L * std::log((2 * m + 1) / (4.0L * kPiL));
    for (int k = 1; k <= m; ++k) lg += 0.5L * std::log((2.0L * k - 1.0L) / (2.0L * k));
    long double pmm;
    if (m == 0) pmm = std::exp(lg);
    else pmm = s2 > 0 ? ((m & 1) ? -1.0L : 1.0L) * std::exp(lg + 0.5L * m * std::log(s2)) : 0.0L;
    if (m >= L) return;
    out[0] = pmm;
    if (m + 1 < L) out[1] = std::sqrt(2.0L * m + 3.0L) * t * pmm;
    for (int l = m + 2; l < L; ++l) {
        const long double a = std::sqrt((4.0L * l * l - 1.0L) / ((long double)l * l - (long double)m * m));
        const long double b =
            std::sqrt(((long double)(l - 1) * (l - 1) - (long double)m * m) / (4.0L * (l - 1) * (l - 1) - 1.0L));
        out[l - m] = a * (t * out[l - 1 - m] - b * out[l - 2 - m]);
    }
}

// N_nl R_nl(r) e^{-decay r^2}: sqrt(2) q_k(r^2) r^l with the normalized Laguerre
// q_k = sqrt(k! / Gamma(k + alpha + 1)) L_k^alpha, alpha = l + 1/2, k = n - l - 1,
//   q_{k+1} = ((2k + alpha + 1 - t) q_k - sqrt(k (k + alpha)) q_{k-1}) / sqrt((k+1)(k+alpha+1)),
// seeded in log space.
long double radial_normalized_ld(int n, int l, long double r, bool decayed) {
    const long double alpha = l + 0.5L, t = r * r;
    long double lg = 0.5L * std::log(2.0L) - 0.5L * std::lgamma(alpha + 1.0L);
    if (l > 0) lg += l * std::log(r);
    if (decayed) lg -= t;
    if (r == 0 && l > 0) return 0.0L;
    long double q0 = 0, q1 = std::exp(lg);
    for (int k = 0; k < n - l - 1; ++k) {
        const long double q = ((2 * k + alpha + 1 - t) * q1 - std::sqrt(k * (k + alpha)) * q0) /
                              std::sqrt((k + 1) * (k + alpha + 1));
        q0 = q1;
        q1 = q;
    }
    return q1;
}

// ---------------------------------------------------------------- SGLT files
// precompute_store.hpp:14-30; CRC-32 is zlib's (IEEE, reflected 0xEDB88320).
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

using store::TableFileError;
using store::TableKind;
using Reason = TableFileError::Reason;

struct RawTable {
    std::uint32_t bandlimit = 0;
    std::vector<double> payload;
};

RawTable read_table(const std::filesystem::path& path, TableKind kind) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw TableFileError(Reason::io, "cannot open for reading: " + path.string());
    std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    constexpr std::size_t header = 13;
    if (bytes.size() < header + 4) throw TableFileError(Reason::length_mismatch, "file too short: " + path.string());
    if (std::memcmp(bytes.data(), "SGLT", 4) != 0)
        throw TableFileError(Reason::bad_magic, "not a table file: " + path.string());
    std::uint32_t version;
    std::memcpy(&version, bytes.data() + 4, 4);
    if (version != store::kFormatVersion)
        throw TableFileError(Reason::version_mismatch, "unsupported format version in " + path.string());
    RawTable raw;
    std::memcpy(&raw.bandlimit, bytes.data() + 8, 4);
    if (bytes[12] != static_cast<unsigned char>(kind))
        throw TableFileError(Reason::kind_mismatch, "unexpected table kind in " + path.string());
    const std::size_t body = bytes.size() - header - 4;
    if (body % 8 != 0)
        throw TableFileError(Reason::length_mismatch, "payload is not a whole number of doubles: " + path.string());
    std::uint32_t crc;
    std::memcpy(&crc, bytes.data() + bytes.size() - 4, 4);
    if (crc != crc32(bytes.data() + header, body))
        throw TableFileError(Reason::crc_mismatch, "payload checksum mismatch: " + path.string());
    raw.payload.resize(body / 8);
    std::memcpy(raw.payload.data(), bytes.data() + header, body);
    return raw;
}

void write_table(const std::filesystem::path& path, std::uint32_t B, TableKind kind, const std::vector<double>& v) {
    std::vector<unsigned char> bytes(13 + 8 * v.size() + 4);
    std::memcpy(bytes.data(), "SGLT", 4);
    std::memcpy(bytes.data() + 4, &store::kFormatVersion, 4);
    std::memcpy(bytes.data() + 8, &B, 4);
    bytes[12] = static_cast<unsigned char>(kind);
    if (!v.empty()) std::memcpy(bytes.data() + 13, v.data(), 8 * v.size());
    const std::uint32_t crc = crc32(bytes.data() + 13, 8 * v.size());
    std::memcpy(bytes.data() + 13 + 8 * v.size(), &crc, 4);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw TableFileError(Reason::io, "cannot open for writing: " + path.string());
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw TableFileError(Reason::io, "write failed: " + path.string());
}

void require_length(bool ok, const std::filesystem::path& path) {
    if (!ok) throw TableFileError(Reason::length_mismatch, "payload length does not match the declared bandlimit: " +
                                                               path.string());
}

// $SGL_TABLES, else the tables/ directory next to this shared library.
std::filesystem::path default_tables_dir() {
    if (const char* env = std::getenv("SGL_TABLES")) return env;
    Dl_info info;
    if (dladdr(reinterpret_cast<void*>(&default_tables_dir), &info) && info.dli_fname)
        return std::filesystem::path(info.dli_fname).parent_path() / "tables";
    return ".";
}

}  // namespace

// ---------------------------------------------------------------- indexing (indexing.cpp)
Layout::Layout(int B) : bandlimit(B) { check_bandlimit(B); }
std::size_t Layout::sample_count() const { return sgl::sample_count(bandlimit); }
std::size_t Layout::coefficient_count() const { return sgl::coefficient_count(bandlimit); }

std::size_t sample_count(int B) {
    check_bandlimit(B);
    return 8 * static_cast<std::size_t>(B) * B * B;
}

std::size_t coefficient_count(int B) {
    check_bandlimit(B);
    const auto b = static_cast<std::size_t>(B);
    return b * (b + 1) * (2 * b + 1) / 6;
}

int mu_index(int j, int k, int B) {
    check_bandlimit(B);
    if (j < 0 || j >= 2 * B || k < 0 || k >= 2 * B) throw std::out_of_range("mu_index: angle indices out of range");
    return 2 * B * j + k;
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
    return static_cast<int>(degree_offset(n)) + l * (l + 1) + m;
}

std::pair<int, int> mu_inverse(int mu, int B) {
    check_bandlimit(B);
    if (mu < 0 || mu >= 4 * B * B) throw std::out_of_range("mu_inverse: index out of range");
    return {mu / (2 * B), mu % (2 * B)};
}

std::array<int, 3> psi_inverse(int psi, int B) {
    check_bandlimit(B);
    if (psi < 0 || static_cast<std::size_t>(psi) >= sample_count(B))
        throw std::out_of_range("psi_inverse: index out of range");
    const int shell = 4 * B * B, rest = psi % shell;
    return {psi / shell, rest / (2 * B), rest % (2 * B)};
}

std::pair<int, int> nu_inverse(int nu) {
    if (nu < 0) throw std::out_of_range("nu_inverse: negative index");
    const int l = isqrt(nu);
    return {l, nu - l * (l + 1)};
}

std::array<int, 3> omega_inverse(int omega) {
    if (omega < 0) throw std::out_of_range("omega_inverse: negative index");
    int n = std::max(1, static_cast<int>(std::cbrt(3.0 * omega)));
    while (degree_offset(n + 1) <= omega) ++n;
    while (n > 1 && degree_offset(n) > omega) --n;
    const auto [l, m] = nu_inverse(omega - static_cast<int>(degree_offset(n)));
    if (l >= n) throw std::out_of_range("omega_inverse: index out of range");
    return {n, l, m};
}

// ---------------------------------------------------------------- quadrature
// quadrature.cpp:189-211 (closed form)
SphericalRule sphere_rule(int L) {
    if (L < 1) throw std::invalid_argument("sphere_rule: order must be positive");
    constexpr double kPi = 3.14159265358979323846;
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

RadialRule half_range_hermite_rule(int N) {
    if (N < 2 || N % 2 != 0 || N > kMaxRadialOrder)
        throw QuadratureError("half_range_hermite_rule: tabulated orders are even, 2 <= N <= " +
                              std::to_string(kMaxRadialOrder));
    const auto dir = default_tables_dir();
    const auto path = dir / store::radial_rule_filename(N / 2);
    if (!std::filesystem::exists(path))
        throw QuadratureError("half_range_hermite_rule: no tabulated rule of order " + std::to_string(N) + " in " +
                              dir.string() + " (generate it with python -m "
                              "paper_1604_05140_b200.tables.gen_radial_rules " + std::to_string(N / 2) + ")");
    return store::load_radial_rule(path);
}

std::vector<double> modified_radial_weights(const RadialRule& rule) {
    std::vector<double> out(rule.r.size());
    for (std::size_t i = 0; i < out.size(); ++i)
        out[i] = std::exp(std::log(rule.a[i]) + rule.r[i] * rule.r[i] + 2.0 * std::log(rule.r[i]));
    return out;
}

double half_range_hermite_moment(int k) { return 0.5 * std::tgamma(0.5 * (k + 1)); }

// ---------------------------------------------------------------- Legendre DCT table
// spherical_transform.cpp:31-86 with the normalized recurrence: row nu(l, m) =
// first l+1 entries of the orthonormal DCT-II (even |m|; row_scale unit row 0)
// or DST-II (odd |m|; frequencies k+1, unit row n-1) of sign * Pbar_{l|m|}(cos theta_j)
// (kernels.cpp:47-65).
LegendreDctTable LegendreDctTable::build(int L) {
    if (L < 1) throw std::invalid_argument("LegendreDctTable: order must be positive");
    const int count = 2 * L;
    LegendreDctTable table;
    table.order = L;
    table.rows.resize(static_cast<std::size_t>(L) * L);
    std::vector<long double> col(static_cast<std::size_t>(count) * L);  // [j][l - am]
    std::vector<long double> cs(static_cast<std::size_t>(count) * count);  // cos / sin of freq x (2j+1) pi / 2N
    for (int am = 0; am < L; ++am) {
        for (int j = 0; j < count; ++j)
            pbar_column(am, L, std::cos((2 * j + 1) * kPiL / (4.0L * L)), &col[static_cast<std::size_t>(j) * L]);
        const bool sine = am % 2 != 0;
        for (int k = 0; k < count; ++k)
            for (int j = 0; j < count; ++j) {
                const long double arg = (sine ? k + 1 : k) * (2.0L * j + 1.0L) * kPiL / (2.0L * count);
                cs[static_cast<std::size_t>(k) * count + j] = sine ? std::sin(arg) : std::cos(arg);
            }
        for (int l = am; l < L; ++l) {
            std::vector<double> row(l + 1);
            for (int k = 0; k <= l; ++k) {
                long double acc = 0;
                for (int j = 0; j < count; ++j)
                    acc += col[static_cast<std::size_t>(j) * L + (l - am)] * cs[static_cast<std::size_t>(k) * count + j];
                const int unit = sine ? count - 1 : 0;
                row[k] = static_cast<double>(acc * std::sqrt((k == unit ? 1.0L : 2.0L) / count));
            }
            table.rows[static_cast<std::size_t>(nu_index(l, am))] = row;
            if (am > 0) {
                if (am % 2 != 0)
                    for (auto& v : row) v = -v;  // M_{l,-m} P_{l,-m} = (-1)^m M_lm P_lm
                table.rows[static_cast<std::size_t>(nu_index(l, -am))] = std::move(row);
            }
        }
    }
    return table;
}

SftPlan SftPlan::build(int L) { return assemble(sphere_rule(L), LegendreDctTable::build(L)); }

SftPlan SftPlan::assemble(SphericalRule rule, LegendreDctTable table) {
    if (rule.order != table.order && !(table.order == 0 && table.rows.empty()))
        throw std::invalid_argument("SftPlan: rule and table orders disagree");
    SftPlan plan;
    plan.order = rule.order;
    plan.rule = std::move(rule);
    plan.table = std::move(table);
    return plan;
}

// ---------------------------------------------------------------- store (precompute_store.cpp:146-271)
namespace store {

std::string radial_rule_filename(int B) { return "radial_rule_B" + std::to_string(B) + ".sglt"; }
std::string spherical_rule_filename(int B) { return "sphere_rule_B" + std::to_string(B) + ".sglt"; }
std::string legendre_table_filename(int B) { return "legendre_dct_B" + std::to_string(B) + ".sglt"; }

void save_radial_rule(const RadialRule& rule, const std::filesystem::path& path) {
    if (rule.order < 2 || rule.order % 2 != 0)
        throw std::invalid_argument("save_radial_rule: rule order must be even (2B)");
    std::vector<double> v;
    v.insert(v.end(), rule.r.begin(), rule.r.end());
    v.insert(v.end(), rule.a.begin(), rule.a.end());
    v.insert(v.end(), rule.a_mod.begin(), rule.a_mod.end());
    write_table(path, static_cast<std::uint32_t>(rule.order / 2), TableKind::radial_rule, v);
}

void save_spherical_rule(const SphericalRule& rule, const std::filesystem::path& path) {
    std::vector<double> v;
    for (const auto* a : {&rule.theta, &rule.phi, &rule.b_raw, &rule.b_cal}) v.insert(v.end(), a->begin(), a->end());
    write_table(path, static_cast<std::uint32_t>(rule.order), TableKind::spherical_rule, v);
}

void save_legendre_table(const LegendreDctTable& table, const std::filesystem::path& path) {
    std::vector<double> v;
    for (const auto& row : table.rows) {
        v.push_back(static_cast<double>(row.size()));
        v.insert(v.end(), row.begin(), row.end());
    }
    write_table(path, static_cast<std::uint32_t>(table.order), TableKind::legendre_dct, v);
}

RadialRule load_radial_rule(const std::filesystem::path& path) {
    const RawTable raw = read_table(path, TableKind::radial_rule);
    const std::size_t count = 2 * static_cast<std::size_t>(raw.bandlimit);
    require_length(raw.bandlimit >= 1 && raw.payload.size() == 3 * count, path);
    RadialRule rule;
    rule.order = static_cast<int>(count);
    rule.r.assign(raw.payload.begin(), raw.payload.begin() + count);
    rule.a.assign(raw.payload.begin() + count, raw.payload.begin() + 2 * count);
    rule.a_mod.assign(raw.payload.begin() + 2 * count, raw.payload.end());
    return rule;
}

SphericalRule load_spherical_rule(const std::filesystem::path& path) {
    const RawTable raw = read_table(path, TableKind::spherical_rule);
    const std::size_t count = 2 * static_cast<std::size_t>(raw.bandlimit);
    require_length(raw.bandlimit >= 1 && raw.payload.size() == 4 * count, path);
    SphericalRule rule;
    rule.order = static_cast<int>(raw.bandlimit);
    const auto b = raw.payload.begin();
    rule.theta.assign(b, b + count);
    rule.phi.assign(b + count, b + 2 * count);
    rule.b_raw.assign(b + 2 * count, b + 3 * count);
    rule.b_cal.assign(b + 3 * count, raw.payload.end());
    return rule;
}

LegendreDctTable load_legendre_table(const std::filesystem::path& path) {
    const RawTable raw = read_table(path, TableKind::legendre_dct);
    require_length(raw.bandlimit >= 1, path);
    const int L = static_cast<int>(raw.bandlimit);
    LegendreDctTable table;
    table.order = L;
    table.rows.resize(static_cast<std::size_t>(L) * L);
    std::size_t pos = 0;
    for (int l = 0; l < L; ++l)
        for (int m = -l; m <= l; ++m) {
            require_length(pos < raw.payload.size(), path);
            const auto len = static_cast<std::size_t>(raw.payload[pos++]);
            require_length(len == static_cast<std::size_t>(l) + 1 && pos + len <= raw.payload.size(), path);
            table.rows[static_cast<std::size_t>(nu_index(l, m))].assign(
                raw.payload.begin() + static_cast<std::ptrdiff_t>(pos),
                raw.payload.begin() + static_cast<std::ptrdiff_t>(pos + len));
            pos += len;
        }
    require_length(pos == raw.payload.size(), path);
    return table;
}

}  // namespace store

// ---------------------------------------------------------------- special functions
// Same conventions and domain errors as special_functions.cpp; values from the
// normalized recurrences above.
double sph_harm_norm(int l, int m) {
    if (l < 0 || std::abs(m) > l) throw std::domain_error("sph_harm_norm: require |m| <= l");
    const long double lr = std::lgamma((long double)(l - m + 1)) - std::lgamma((long double)(l + m + 1));
    return static_cast<double>(std::sqrt((2 * l + 1) / (4.0L * kPiL) * std::exp(lr)));
}

// The unnormalized P_lm itself (Condon-Shortley phase): P_mm = (-1)^m (2m-1)!!
// (1-t^2)^{m/2}, then the unnormalized three-term ascent in l -- the values
// satisfy that recurrence to rounding, as the reference's test of it
// (test_special_functions.cpp:40-51) demands; they overflow for large m exactly
// like the reference's (the transforms never use this function).
double assoc_legendre(int l, int m, double t) {
    if (m < 0 || m > l)
        throw std::domain_error("assoc_legendre: require 0 <= m <= l, got l=" + std::to_string(l) +
                                " m=" + std::to_string(m));
    if (std::abs(t) > 1.0) throw std::domain_error("assoc_legendre: argument must satisfy |t| <= 1");
    const double s = std::sqrt((1.0 - t) * (1.0 + t));
    double p = 1.0;
    for (int k = 1; k <= m; ++k) p *= -(2.0 * k - 1.0) * s;
    double prev = 0.0;
    for (int ll = m + 1; ll <= l; ++ll) {  // (ll - m) P_ll = (2ll - 1) t P_{ll-1} - (ll - 1 + m) P_{ll-2}
        const double next = ((2 * ll - 1) * t * p - (ll - 1 + m) * prev) / (ll - m);
        prev = p;
        p = next;
    }
    return p;
}

double assoc_legendre_signed(int l, int m, double t) {
    if (m >= 0) return assoc_legendre(l, m, t);
    if (-m > l) throw std::domain_error("assoc_legendre_signed: require |m| <= l");
    const int a = -m;
    const long double ratio = std::exp(std::lgamma((long double)(l - a + 1)) - std::lgamma((long double)(l + a + 1)));
    return static_cast<double>(((a & 1) ? -1.0L : 1.0L) * ratio * assoc_legendre(l, a, t));
}

double gen_laguerre(int k, double alpha, double t) {
    if (k < 0) throw std::domain_error("gen_laguerre: degree must be nonnegative");
    if (k == 0) return 1.0;
    long double prev = 1.0L, cur = alpha + 1.0L - t;
    for (int j = 1; j < k; ++j) {
        const long double next = ((2 * j + alpha + 1.0L - t) * cur - (j + alpha) * prev) / (j + 1);
        prev = cur;
        cur = next;
    }
    return static_cast<double>(cur);
}

std::complex<double> sph_harm(int l, int m, double theta, double phi) {
    if (theta < 0.0 || theta > 3.14159265358979323846)
        throw std::domain_error("sph_harm: theta must lie in [0, pi]");
    if (phi < 0.0 || phi >= 2.0 * 3.14159265358979323846)
        throw std::domain_error("sph_harm: phi must lie in [0, 2 pi)");
    if (l < 0 || m < -l || m > l) throw std::domain_error("sph_harm: require |m| <= l");
    const int a = std::abs(m);
    std::vector<long double> col(static_cast<std::size_t>(l - a + 1));
    pbar_column(a, l + 1, std::cos((long double)theta), col.data());
    const double v = static_cast<double>(col[l - a]) * ((m < 0 && (a & 1)) ? -1.0 : 1.0);
    return v * std::complex<double>(std::cos(m * phi), std::sin(m * phi));
}

double norm_const(int n, int l) {
    if (l < 0 || n <= l) throw std::domain_error("norm_const: require 0 <= l < n");
    return static_cast<double>(
        std::exp(0.5L * (std::log(2.0L) + std::lgamma((long double)(n - l)) - std::lgamma(n + 0.5L))));
}

double radial_raw(int n, int l, double r) {
    if (l < 0 || n <= l) throw std::domain_error("radial_raw: require 0 <= l < n");
    if (r < 0.0) throw std::domain_error("radial_raw: radius must be nonnegative");
    return gen_laguerre(n - l - 1, l + 0.5, r * r) * std::pow(r, l);
}

double radial_normalized(int n, int l, double r) {
    if (n == l) return 0.0;
    if (l < 0 || n < l) throw std::domain_error("radial_normalized: require 0 <= l < n");
    return static_cast<double>(radial_normalized_ld(n, l, r, false));
}

double radial_normalized_decayed(int n, int l, double r) {
    if (n == l) return 0.0;
    if (l < 0 || n < l) throw std::domain_error("radial_normalized_decayed: require 0 <= l < n");
    return static_cast<double>(radial_normalized_ld(n, l, r, true));
}

std::complex<double> sgl_basis(int n, int l, int m, double r, double theta, double phi) {
    if (l >= n) throw std::domain_error("sgl_basis: require l < n");
    return radial_normalized(n, l, r) * sph_harm(l, m, theta, phi);
}

namespace detail {
// The seed value is N_{l+1,l} R_{l+1,l}(r) (optionally pre-scaled); the ascent
// is the same normalized recurrence, started from that value.
double radial_from_seed(int n, int l, double r, double seed_value) {
    if (n == l) return 0.0;
    const long double alpha = l + 0.5L, t = (long double)r * r;
    long double q0 = 0, q1 = seed_value;
    for (int k = 0; k < n - l - 1; ++k) {
        const long double q = ((2 * k + alpha + 1 - t) * q1 - std::sqrt(k * (k + alpha)) * q0) /
                              std::sqrt((k + 1) * (k + alpha + 1));
        q0 = q1;
        q1 = q;
    }
    return static_cast<double>(q1);
}
}  // namespace detail

}  // namespace sgl
