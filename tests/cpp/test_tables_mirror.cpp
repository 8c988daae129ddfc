// Host-only check of the plan-table surface of the C++ mirror (no GPU needed:
// the device plan is created lazily).  Usage: test_tables_mirror <dir> <B> <out_dir>
//   <dir>      SGLT kinds 1-3 written by the REFERENCE (oracle/_ref, ref_save_tables)
//   <out_dir>  where the mirror re-saves them (for a byte comparison by the caller)
// Checks TransformPlan::from_tables (kinds 1, 2, 3; sgl_transform.cpp:98-102),
// the 4-argument assemble and its order validation (:52-63), and
// LegendreDctTable::build against the reference's rows.  Prints
// "max_row_err <x>" and exits nonzero on a failed check.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "sgl/precompute_store.hpp"
#include "sgl/sgl_transform.hpp"

using namespace sgl;

int main(int argc, char** argv) {
    if (argc != 4) return 2;
    const std::filesystem::path dir = argv[1], out = argv[3];
    const int B = std::atoi(argv[2]);
    int fails = 0;
    auto check = [&](bool ok, const char* what) {
        if (!ok) {
            std::printf("FAIL %s\n", what);
            ++fails;
        }
    };
    const TransformPlan plan = TransformPlan::from_tables(dir, B);
    check(plan.bandlimit == B && plan.radial.order == 2 * B, "radial rule order");
    check(plan.sphere.order == B && plan.sphere.table.order == B, "spherical orders");
    check(plan.sphere.table.rows.size() == static_cast<std::size_t>(B) * B, "table rows loaded (kind 3)");
    const SphericalRule closed = sphere_rule(B);
    check(plan.sphere.rule.b_cal == closed.b_cal && plan.sphere.rule.theta == closed.theta, "kind 2 == closed form");
    // the mirror's own DCT rows against the reference's (relative to the row's scale)
    const LegendreDctTable mine = LegendreDctTable::build(B);
    double worst = 0.0;
    for (int l = 0; l < B; ++l)
        for (int m = -l; m <= l; ++m) {
            const auto& a = mine.rows[nu_index(l, m)];
            const auto& b = plan.sphere.table.rows[nu_index(l, m)];
            if (a.size() != b.size()) {
                check(false, "row length");
                continue;
            }
            for (std::size_t k = 0; k < a.size(); ++k) worst = std::max(worst, std::abs(a[k] - b[k]));
        }
    std::printf("max_row_err %.3e\n", worst);
    // assemble's validation (sgl_transform.cpp:52-63), messages included
    try {
        LegendreDctTable wrong;
        wrong.order = B + 1;
        TransformPlan::assemble(B, plan.radial, plan.sphere.rule, wrong);
        check(false, "table order mismatch must throw");
    } catch (const std::invalid_argument& e) {
        check(std::string(e.what()) == "TransformPlan: spherical tables must have order B", "message");
    }
    try {
        TransformPlan::assemble(B, plan.radial, sphere_rule(B + 1), mine);
        check(false, "rule order mismatch must throw");
    } catch (const std::invalid_argument&) {
    }
    const TransformPlan p4 = TransformPlan::assemble(B, plan.radial, plan.sphere.rule, mine);
    check(p4.m_norm.size() == static_cast<std::size_t>(B) * B && p4.exp_neg_r2.size() == 2u * B, "derived vectors");
    // re-save through the mirror's writers
    std::filesystem::create_directories(out);
    store::save_radial_rule(plan.radial, out / store::radial_rule_filename(B));
    store::save_spherical_rule(plan.sphere.rule, out / store::spherical_rule_filename(B));
    store::save_legendre_table(plan.sphere.table, out / store::legendre_table_filename(B));
    // corrupted file -> TableFileError with the right reason
    try {
        store::load_legendre_table(out / store::radial_rule_filename(B));
        check(false, "kind mismatch must throw");
    } catch (const store::TableFileError& e) {
        check(e.reason == store::TableFileError::Reason::kind_mismatch, "kind_mismatch reason");
    }
    return fails;
}
