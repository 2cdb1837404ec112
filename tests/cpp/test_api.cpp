// C++ API test of the B200-native spmvcomp: the reference's worked examples and
// acceptance criteria (SPEC.md, cited per check) run through the reference's own C++
// interface, with every operation executing on the GPU.  Exit code 0 = all passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "spmvcomp/compress.hpp"
#include "spmvcomp/ell.hpp"
#include "spmvcomp/errors.hpp"
#include "spmvcomp/kernels.hpp"
#include "spmvcomp/perf_model.hpp"
#include "spmvcomp/solver.hpp"
#include "spmvcomp/stencil.hpp"
#include "spmvcomp_b200/device.hpp"

using namespace spmvcomp;

static int g_failed = 0, g_checks = 0;
#define CHECK(...)                                                            \
    do {                                                                      \
        g_checks++;                                                           \
        if (!(__VA_ARGS__)) {                                                   \
            g_failed++;                                                       \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__);     \
        }                                                                     \
    } while (0)
template <class E, class F>
static bool throws(F f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

static StencilMatrix fig_matrix() {  // the figure's row as row 50
    std::vector<std::vector<std::pair<std::int32_t, double>>> rows(66);
    for (int i = 0; i < 66; i++) rows[i] = {{i, 26.0}};
    rows[50] = {{45, -1.0}, {49, -1.0}, {50, 26.0}, {51, -1.0}, {65, -1.0}};
    return stencil_from_rows(66, rows);
}

static std::vector<std::vector<double>> dense(const GridSpec& g) {  // brute-force oracle of SPEC.md:216,269
    const int n = (int)g.rows();
    std::vector<std::vector<double>> a(n, std::vector<double>(n, 0.0));
    for (int iz = 0; iz < g.nz; iz++) for (int iy = 0; iy < g.ny; iy++) for (int ix = 0; ix < g.nx; ix++)
        for (int dz = -1; dz <= 1; dz++) for (int dy = -1; dy <= 1; dy++) for (int dx = -1; dx <= 1; dx++) {
            const int x = ix + dx, y = iy + dy, z = iz + dz;
            if (x < 0 || x >= g.nx || y < 0 || y >= g.ny || z < 0 || z >= g.nz) continue;
            const int i = (int)g.node(ix, iy, iz), j = (int)g.node(x, y, z);
            a[i][j] = i == j ? 26.0 : -1.0;
        }
    return a;
}

int main() {
    // ---- generator
    {
        const StencilMatrix m1 = generate_matrix(GridSpec{1, 1, 1});
        CHECK(m1.n == 1 && m1.nnz() == 1 && m1.cols[0] == 0 && m1.vals[0] == 26.0);
        const StencilMatrix m2 = generate_matrix(GridSpec{2, 2, 2});
        CHECK(m2.n == 8);
        for (int i = 0; i < 8; i++) {
            double s = 0;
            for (double v : m2.row_vals(i)) s += v;
            CHECK(m2.row_nnz(i) == 8 && s == 19.0);
        }
        const GridSpec g4{4, 4, 4};
        const StencilMatrix m4 = generate_matrix(g4);
        const int i = (int)g4.node(1, 1, 1);
        double s = 0;
        for (double v : m4.row_vals(i)) s += v;
        CHECK(m4.row_nnz(i) == 27 && s == 0.0);
        CHECK(is_symmetric(m4) && m4.grid == g4);
        CHECK(m4.nnz() == 10 * 10 * 10);
        CHECK(throws<std::invalid_argument>([] { generate_matrix(GridSpec{0, 1, 1}); }));
        CHECK(throws<std::invalid_argument>([] { generate_matrix(GridSpec{100000, 100000, 100000}); }));
    }
    // ---- vectors
    {
        CHECK(make_test_vector(3, VectorKind::ones) == (Vector{1, 1, 1}));
        CHECK(make_test_vector(3, VectorKind::linear) == (Vector{0, 1, 2}));
        const Vector a = make_test_vector(4, VectorKind::random, 7), b = make_test_vector(4, VectorKind::random, 7);
        CHECK(a == b && a[0] >= 0.0 && a[0] < 1.0);
        CHECK(throws<std::invalid_argument>([] { make_test_vector(4, VectorKind::random); }));
    }
    // ---- the figure row through every format
    {
        const StencilMatrix m = fig_matrix();
        const EllMatrix e = to_ell(m);
        CHECK(e.width == 5);
        CHECK((std::vector<double>(e.values.begin() + 250, e.values.begin() + 255) == std::vector<double>{-1, -1, 26, -1, -1}));
        CHECK((std::vector<std::int32_t>(e.columns.begin() + 250, e.columns.begin() + 255) == std::vector<std::int32_t>{45, 49, 50, 51, 65}));
        const VtCompressedMatrix vt = compress_values(m);
        CHECK((vt.table.entries == std::vector<double>{-1.0, 26.0}));
        CHECK((std::vector<std::int32_t>(vt.sorted_columns.begin() + 250, vt.sorted_columns.begin() + 255) == std::vector<std::int32_t>{45, 49, 51, 65, 50}));
        CHECK(vt.ends[100] == 4 && vt.ends[101] == 5);
        const PatternCompressedMatrix pc = compress_patterns(m, false);
        const DisplacementPattern& p = pc.patterns[pc.row_pattern[50]];
        CHECK((p.displacements == std::vector<std::int32_t>{-5, -1, 1, 15, 0}) && (p.ends == std::vector<std::int32_t>{4, 5}));
        const Vector ones(66, 1.0);
        CHECK(spmv(e, ones)[50] == 22.0 && spmv(vt, ones)[50] == 22.0 && spmv(pc, ones)[50] == 22.0);
        CHECK(decompress(vt) == m && decompress(pc) == m && to_stencil(e) == m);
    }
    // ---- 1x1 examples
    {
        const StencilMatrix m = generate_matrix(GridSpec{1, 1, 1});
        CHECK(spmv(to_ell(m), Vector{2.0}) == Vector{52.0});
        CHECK(spmv(compress_values(m), Vector{1.0}) == Vector{26.0});
        CHECK(spmv(compress_patterns(m, true), Vector{-1.0}) == Vector{-26.0});
        const VtCompressedMatrix vt = compress_values(m);
        CHECK(vt.table.entries == std::vector<double>{26.0} && vt.sorted_columns == std::vector<std::int32_t>{0} && vt.ends == std::vector<std::int32_t>{1});
    }
    // ---- pattern counts, round trips, cross-format agreement
    for (int nx = 1; nx <= 5; nx++) for (int ny = 1; ny <= 4; ny++) for (int nz = 1; nz <= 4; nz++) {
        const GridSpec g{nx, ny, nz};
        const StencilMatrix m = generate_matrix(g);
        const EllMatrix e = to_ell(m);
        const VtCompressedMatrix vt = compress_values(m);
        const PatternCompressedMatrix pc = compress_patterns(m, true);
        CHECK((int)pc.patterns.size() == std::min(nx, 3) * std::min(ny, 3) * std::min(nz, 3));
        validate(vt);
        validate(pc);
        CHECK(decompress(vt) == m && decompress(pc) == m && to_stencil(e) == m);
        CHECK(compress_patterns(m, true) == pc);  // byte-identical recompression
        if (m.n >= 2) CHECK((pc.table.entries == std::vector<double>{-1.0, 26.0}));
        const auto a = dense(g);
        for (std::uint64_t seed = 1; seed <= 2; seed++) {
            const Vector x = make_test_vector(m.n, VectorKind::random, seed);
            const Vector ye = spmv(e, x), yv = spmv(vt, x), yp = spmv(pc, x);
            for (int i = 0; i < m.n; i++) {
                double ref = 0, scale = 0;
                for (int j = 0; j < m.n; j++) { ref += a[i][j] * x[j]; scale += std::fabs(a[i][j] * x[j]); }
                CHECK(std::fabs(ye[i] - ref) <= 1e-13 * scale && std::fabs(yv[i] - ref) <= 1e-13 * scale &&
                      std::fabs(yp[i] - ref) <= 1e-13 * scale);
            }
        }
    }
    // ---- A*ones, row ranges, errors (kernels.hpp:27-29)
    {
        const StencilMatrix m = generate_matrix(GridSpec{6, 5, 4});
        const PatternCompressedMatrix pc = compress_patterns(m, false);
        const EllMatrix e = to_ell(m);
        const Vector y1 = spmv(pc, Vector(m.n, 1.0));
        for (double v : y1) CHECK(v >= 0.0);
        CHECK(y1[GridSpec{6, 5, 4}.node(2, 2, 2)] == 0.0);
        const Vector x = make_test_vector(m.n, VectorKind::random, 7);
        const Vector full = spmv(pc, x);
        Vector y(m.n, 123.0);
        unchecked::spmv_rows(pc, x, y, 0, 17);
        unchecked::spmv_rows(pc, x, y, 40, m.n);
        bool ok = true;
        for (int i = 0; i < m.n; i++) ok = ok && (i >= 17 && i < 40 ? y[i] == 123.0 : !std::memcmp(&y[i], &full[i], 8));
        CHECK(ok);
        Vector ye(m.n, 0.0);
        unchecked::spmv_rows(e, x, ye, 0, m.n);
        CHECK(ye == spmv(e, x));
        CHECK(throws<std::invalid_argument>([&] { spmv(pc, Vector(5, 1.0)); }));
        CHECK(throws<std::invalid_argument>([&] { spmv(e, Vector(5, 1.0)); }));
        PatternCompressedMatrix bad = pc;
        bad.row_pattern[3] = 999;
        CHECK(throws<IntegrityError>([&] { spmv(bad, x); }));
        CHECK(throws<IntegrityError>([&] { validate(bad); }));
        VtCompressedMatrix vt = compress_values(m);
        vt.ends[1] = 0;
        CHECK(throws<IntegrityError>([&] { validate(vt); }));
        CHECK(throws<IntegrityError>([&] { decompress(vt); }));
        std::vector<std::vector<std::pair<std::int32_t, double>>> rows(300);
        for (int i = 0; i < 300; i++) rows[i] = {{i, i + 1.0}};
        const StencilMatrix many = stencil_from_rows(300, rows);
        CHECK(throws<TableOverflowError>([&] { compress_values(many); }));
        CHECK(throws<TableOverflowError>([&] { compress_patterns(many, false); }));
        CHECK(scan_value_table(many, 300).size() == 300);
        CHECK(throws<std::invalid_argument>([] { stencil_from_rows(2, {{{1, 1.0}, {0, 1.0}}, {{1, 1.0}}}); }));
    }
    // ---- byte model
    {
        CHECK(format_cost(MatrixFormat::ell, 27, 2).bytes_per_row == 324.0);
        CHECK(format_cost(MatrixFormat::vt, 27, 2).bytes_per_row == 116.0);
        CHECK(format_cost(MatrixFormat::pattern, 27, 2).bytes_per_row == 12.0);
        CHECK(format_cost(MatrixFormat::pattern_with_values, 27, 2).bytes_per_row == 4.0);
        const FormatCost ell = format_cost(MatrixFormat::ell, 27, 2);
        CHECK(std::fabs(required_bandwidth(11.6e9, ell) - 69.6e9) < 1.0);
        CHECK(std::fabs(roofline(ell, MachineSpec{}).predicted_flops - 12.5e9) < 1.0);
        CHECK(std::fabs(roofline(format_cost(MatrixFormat::vt, 27, 2), MachineSpec{}).predicted_flops / 1e9 - 34.9) < 0.05);
        CHECK(std::fabs(roofline(format_cost(MatrixFormat::pattern, 27, 2), MachineSpec{}).predicted_flops / 1e9 - 337.5) < 1e-6);
        const StencilMatrix m = generate_matrix(GridSpec{32, 32, 32});
        CHECK(measured_cost(to_ell(m)).bytes_per_row == 324.0);
        const double pv = measured_cost(compress_patterns(m, true)).bytes_per_row;
        CHECK(pv > 4.0 && pv < 4.08);
        CHECK(measured_cost(compress_values(m)).bytes_per_row == 116.0);
        CHECK(std::string(format_name(MatrixFormat::pattern_with_values)) == "pattern-values" && parse_format("vt") == MatrixFormat::vt);
        // model_table / model_table_csv / model_table_json (inc/perf_model.hpp:82-95)
        MachineSpec slow;
        slow.peak_flops = 100e9;  // below the 337.5 Gflops the bandwidth would allow for `pattern`
        const std::vector<ModelRow> rows = model_table({MatrixFormat::ell, MatrixFormat::vt, MatrixFormat::pattern}, 27, 2, slow);
        CHECK(rows.size() == 3 && rows[0].format == MatrixFormat::ell && rows[0].cost.bytes_per_row == 324.0);
        CHECK(std::fabs(rows[0].estimate.predicted_flops - 12.5e9) < 1.0 && rows[0].estimate.limiting_resource == LimitingResource::bandwidth);
        CHECK(rows[2].estimate.predicted_flops == 100e9 && rows[2].estimate.limiting_resource == LimitingResource::compute);
        const std::string csv = model_table_csv(rows);
        CHECK(csv.rfind("format,bytes_per_row,bytes_per_flop,predicted_gflops,limiting_resource\n", 0) == 0);
        CHECK(csv.find("ell,324,6,12.5,bandwidth\n") != std::string::npos && csv.find("pattern,12,") != std::string::npos &&
              csv.find(",100,compute\n") != std::string::npos);
        const std::string js = model_table_json(rows);
        CHECK(js.front() == '[' && js.find("\"format\": \"vt\"") != std::string::npos && js.find("\"limiting_resource\": \"compute\"") != std::string::npos);
        ModelOptions with_x;
        with_x.include_input_vector = true;
        CHECK(model_table({MatrixFormat::pattern_with_values}, 27, 2, MachineSpec{}, with_x)[0].cost.bytes_per_row == 12.0);
    }
    // ---- the CG caller (acceptance criterion 8)
    {
        CHECK(dot(Vector{1, 2}, Vector{3, 4}) == 11.0);
        CHECK(dot(Vector(1000, 1.0), Vector(1000, 1.0)) == 1000.0);
        CHECK(waxpby(2, Vector{1, 1}, 3, Vector{1, 2}) == (Vector{5, 8}));
        CHECK(waxpby(1, Vector{1, 1}, 0, Vector{1, 2}) == (Vector{1, 1}) && waxpby(0, Vector{1, 1}, 1, Vector{1, 2}) == (Vector{1, 2}));
        CHECK(throws<std::invalid_argument>([] { dot(Vector{1}, Vector{1, 2}); }));
        const StencilMatrix one = generate_matrix(GridSpec{1, 1, 1});
        auto [x1, r1] = cg_solve(one, Vector{52.0});
        CHECK(x1 == Vector{2.0} && r1.iterations == 1 && r1.converged);
        const StencilMatrix m = generate_matrix(GridSpec{16, 16, 16});
        const Vector b = spmv(to_ell(m), Vector(m.n, 1.0));
        int its[3];
        Vector xs[3];
        int k = 0;
        for (SpmvBackend be : {SpmvBackend::ell, SpmvBackend::vt, SpmvBackend::pattern}) {
            CgConfig cfg;
            cfg.backend = be;
            auto [x, rep] = cg_solve(m, b, cfg);
            its[k] = rep.iterations;
            xs[k] = x;
            double worst = 0;
            for (double v : x) worst = std::max(worst, std::fabs(v - 1.0));
            CHECK(rep.converged && rep.final_residual() <= 1e-8 && worst <= 1e-6);
            CHECK((int)rep.residual_history.size() == rep.iterations + 1 && rep.residual_history[0] == 1.0);
            CHECK(rep.flops_total == (std::int64_t)rep.iterations * (2 * m.nnz() + 12 * (std::int64_t)m.n));
            CHECK(rep.per_op.at("spmv").calls == rep.iterations && rep.per_op.at("dot").calls == 3 * rep.iterations);
            k++;
        }
        CHECK(its[0] == its[1] && its[1] == its[2]);
        double d = 0;
        for (int i = 0; i < m.n; i++) d = std::max({d, std::fabs(xs[0][i] - xs[1][i]), std::fabs(xs[0][i] - xs[2][i])});
        CHECK(d <= 1e-9);
        CgConfig one_it;
        one_it.max_iterations = 1;
        CHECK(!cg_solve(m, b, one_it).second.converged);
        // SymGS preconditioner (inc/solver.hpp:17-28): fewer iterations, same solution, analytic flop count
        CgConfig pre;
        pre.symgs_sweeps = 1;
        auto [xp, rp] = cg_solve(m, b, pre);
        double worst = 0;
        for (double v : xp) worst = std::max(worst, std::fabs(v - 1.0));
        CHECK(rp.converged && rp.iterations < its[0] && worst <= 1e-6);
        CHECK(rp.per_op.at("precond").calls == rp.iterations && rp.per_op.at("precond").flops == rp.iterations * symgs_flops(m.nnz()));
        CHECK(rp.flops_total == (std::int64_t)rp.iterations * (2 * m.nnz() + 12 * (std::int64_t)m.n) + rp.per_op.at("precond").flops);
        StencilMatrix no_grid = m;  // without provenance the device sweep has no schedule
        no_grid.grid = GridSpec{0, 0, 0};
        CHECK(throws<std::invalid_argument>([&] { cg_solve(no_grid, b, pre); }));
        pre.symgs_sweeps = -1;
        CHECK(throws<std::invalid_argument>([&] { cg_solve(m, b, pre); }));
    }
    // ---- symgs_sweep (inc/kernels.hpp:44-48)
    {
        const StencilMatrix one = generate_matrix(GridSpec{1, 1, 1});
        Vector x{0.0};
        symgs_sweep(one, x, Vector{52.0});
        CHECK(x[0] == 2.0);  // exact solve of the 1x1 system
        const StencilMatrix m = generate_matrix(GridSpec{3, 3, 3});
        const Vector b = spmv(to_ell(m), Vector(m.n, 1.0));
        Vector y(m.n, 0.0), y2(m.n, 0.0);
        symgs_sweep(m, y, b);
        symgs_sweep(m, y2, b);
        CHECK(std::memcmp(y.data(), y2.data(), y.size() * sizeof(double)) == 0);  // deterministic
        const Vector ay = spmv(to_ell(m), y);
        double r0 = 0, r1 = 0;
        for (int i = 0; i < m.n; i++) r0 += b[i] * b[i], r1 += (b[i] - ay[i]) * (b[i] - ay[i]);
        CHECK(r1 < r0);  // the residual norm decreases
        Vector shortx(3, 0.0);
        CHECK(throws<std::invalid_argument>([&] { symgs_sweep(m, shortx, b); }));
        StencilMatrix z = stencil_from_rows(2, {{{0, 1.0}}, {{0, 1.0}}});  // row 1 has no diagonal
        z.grid = GridSpec{2, 1, 1};
        Vector zx(2, 0.0);
        CHECK(throws<std::invalid_argument>([&] { symgs_sweep(z, zx, Vector(2, 1.0)); }));
    }
    // ---- device-resident use: generate and compress on the GPU, many SpMVs, one download
    {
        using namespace spmvcomp::b200;
        const GridSpec g{64, 48, 40};
        const DeviceMatrix csr = DeviceMatrix::generate(g);
        const DeviceMatrix pc = csr.compress_patterns(true), ell = csr.to_ell();
        DeviceVector x(g.rows()), y(g.rows()), y2(g.rows());
        x.fill(VectorKind::random, 7, -1.0, 1.0);
        for (int rep = 0; rep < 3; rep++) spmvcomp::b200::spmv_rows(pc, x, y, 0, (std::int32_t)g.rows());
        spmvcomp::b200::spmv_rows(ell, x, y2, 0, (std::int32_t)g.rows());
        const Vector a = y.download(), b = y2.download(), xs = x.download();
        const Vector ref = spmv(pc.download_pattern(), xs);
        CHECK(!std::memcmp(a.data(), ref.data(), a.size() * 8));
        double worst = 0;
        for (std::size_t i = 0; i < a.size(); i++) worst = std::max(worst, std::fabs(a[i] - b[i]));
        CHECK(worst <= 1e-12 * 52.0);
        CHECK(pc.info().n_patterns == 27 && pc.info().kernel_plan == 1);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
