// Host-only checks of include/spmvcomp/io.hpp (stencil.hpp:61-64).  No GPU needed.
//   test_io <dir>
// <dir> holds files written by the Python restatement (oracle/serial.py): stencil.bin, ell.bin, vt.bin, pattern.bin,
// pattern_values.bin.  Each is loaded, checked against serialized_size, saved again as <name>.out (tests/test_io.py
// compares the bytes), and the matrix is exported to <dir>/matrix.mtx.  Then the error paths.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "spmvcomp/io.hpp"

namespace fs = std::filesystem;
using namespace spmvcomp;

static int checks = 0, failed = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        checks++;                                                            \
        if (!(cond)) {                                                       \
            failed++;                                                        \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
        }                                                                    \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<char> slurp(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    return std::vector<char>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}
static void spit(const fs::path& p, const std::vector<char>& b) {
    std::ofstream out(p, std::ios::binary | std::ios::trunc);
    out.write(b.data(), (std::streamsize)b.size());
}

int main(int argc, char** argv) {
    if (argc != 2) {
        std::fprintf(stderr, "usage: test_io <dir>\n");
        return 2;
    }
    const fs::path dir = argv[1];

    // ---- files of the Python restatement: load, size, save again ----
    CHECK(file_kind(dir / "stencil.bin") == FileKind::stencil);
    CHECK(file_kind(dir / "ell.bin") == FileKind::ell);
    CHECK(file_kind(dir / "vt.bin") == FileKind::vt);
    CHECK(file_kind(dir / "pattern.bin") == FileKind::pattern);
    const StencilMatrix m = load_stencil(dir / "stencil.bin");
    const EllMatrix e = load_ell(dir / "ell.bin");
    const VtCompressedMatrix v = load_vt(dir / "vt.bin");
    const PatternCompressedMatrix p = load_pattern(dir / "pattern.bin");
    const PatternCompressedMatrix pv = load_pattern(dir / "pattern_values.bin");
    CHECK(serialized_size(m) == fs::file_size(dir / "stencil.bin"));
    CHECK(serialized_size(e) == fs::file_size(dir / "ell.bin"));
    CHECK(serialized_size(v) == fs::file_size(dir / "vt.bin"));
    CHECK(serialized_size(p) == fs::file_size(dir / "pattern.bin"));
    CHECK(serialized_size(pv) == fs::file_size(dir / "pattern_values.bin"));
    CHECK(!p.values_in_pattern && pv.values_in_pattern);
    CHECK(p.patterns == pv.patterns && p.row_pattern == pv.row_pattern);
    // per-row ends are the only difference between the two pattern files: 8-byte prefix + n * m * 4 bytes
    CHECK(serialized_size(p) - serialized_size(pv) == 8 + (std::uint64_t)p.n * (std::uint64_t)p.table.size() * 4);
    CHECK(m.n == e.n && m.n == v.n && m.n == p.n && m.nnz() == e.nnz && m.nnz() == v.nnz() && m.nnz() == p.nnz());
    CHECK(m.grid.rows() == m.n);
    // byte accounting: the ELL file is 16 + 16 + 2 * 8 + 12 * n * width bytes
    CHECK(serialized_size(e) == 48 + 12ull * (std::uint64_t)e.n * (std::uint64_t)e.width);
    CHECK(serialized_size(v) == 16 + 8 + 3 * 8 + 8 * v.table.entries.size() + 4ull * (std::uint64_t)v.n * (std::uint64_t)(v.width + v.table.size()));
    save(m, dir / "stencil.bin.out");
    save(e, dir / "ell.bin.out");
    save(v, dir / "vt.bin.out");
    save(p, dir / "pattern.bin.out");
    save(pv, dir / "pattern_values.bin.out");
    CHECK(load_stencil(dir / "stencil.bin.out") == m);
    CHECK(load_ell(dir / "ell.bin.out") == e);
    CHECK(load_vt(dir / "vt.bin.out") == v);
    CHECK(load_pattern(dir / "pattern.bin.out") == p);
    CHECK(load_pattern(dir / "pattern_values.bin.out") == pv);

    // ---- Matrix Market: export (lower triangle), import mirrors it back ----
    write_matrix_market(m, dir / "matrix.mtx");
    const StencilMatrix back = read_matrix_market(dir / "matrix.mtx");
    CHECK(back == m);
    {
        StencilMatrix ns;  // [[1, 2], [0, 3]]: not symmetric
        ns.n = 2, ns.row_start = {0, 2, 3}, ns.cols = {0, 1, 1}, ns.vals = {1.0, 2.0, 3.0};
        CHECK(throws<std::invalid_argument>([&] { write_matrix_market(ns, dir / "ns.mtx"); }));
        save(ns, dir / "ns.bin");
        CHECK(load_stencil(dir / "ns.bin") == ns);
        std::ofstream(dir / "general.mtx") << "%%MatrixMarket matrix coordinate real general\n% comment\n2 2 3\n2 2 3\n1 2 2\n1 1 1\n";
        CHECK(read_matrix_market(dir / "general.mtx") == ns);
        std::ofstream(dir / "dup.mtx") << "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n";
        CHECK(throws<IoError>([&] { read_matrix_market(dir / "dup.mtx"); }));
        std::ofstream(dir / "array.mtx") << "%%MatrixMarket matrix array real general\n1 1\n1\n";
        CHECK(throws<IoError>([&] { read_matrix_market(dir / "array.mtx"); }));
        std::ofstream(dir / "short.mtx") << "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n";
        CHECK(throws<IoError>([&] { read_matrix_market(dir / "short.mtx"); }));
    }

    // ---- the figure's row as a one-row structure: sizes by hand ----
    {
        VtCompressedMatrix f;
        f.n = 1, f.width = 5;
        f.table.entries = {-1.0, 26.0};
        f.sorted_columns = {45, 49, 51, 65, 50};
        f.ends = {4, 5};
        CHECK(serialized_size(f) == 16 + 8 + (8 + 16) + (8 + 20) + (8 + 8));
        save(f, dir / "figure_vt.bin");
        CHECK(fs::file_size(dir / "figure_vt.bin") == serialized_size(f) && load_vt(dir / "figure_vt.bin") == f);
        PatternCompressedMatrix g;
        g.n = 1;
        g.table.entries = {-1.0, 26.0};
        g.patterns.push_back({{-5, -1, 1, 15, 0}, {4, 5}});
        g.row_pattern = {0};
        g.values_in_pattern = true;
        CHECK(serialized_size(g) == 16 + 4 + (8 + 16) + 8 + (8 + 20) + (8 + 8) + (8 + 4) + 1);
        save(g, dir / "figure_pattern.bin");
        CHECK(load_pattern(dir / "figure_pattern.bin") == g);
        g.values_in_pattern = false;
        CHECK(serialized_size(g) == 16 + 4 + (8 + 16) + 8 + (8 + 20) + (8 + 8) + (8 + 4) + 1 + (8 + 8));
        save(g, dir / "figure_pattern_rows.bin");
        CHECK(fs::file_size(dir / "figure_pattern_rows.bin") == serialized_size(g) && load_pattern(dir / "figure_pattern_rows.bin") == g);
        g.row_pattern = {3};  // no such pattern: nothing may be written
        CHECK(throws<IntegrityError>([&] { save(g, dir / "never.bin"); }));
        CHECK(!fs::exists(dir / "never.bin"));
        EllMatrix one;  // 1x1x1: width 1, [[26.0]], [[0]]
        one.n = 1, one.width = 1, one.nnz = 1, one.values = {26.0}, one.columns = {0};
        CHECK(serialized_size(one) == 48 + 12);
        save(one, dir / "one.bin");
        CHECK(load_ell(dir / "one.bin") == one);
    }

    // ---- error paths ----
    const std::vector<char> good = slurp(dir / "pattern.bin");
    CHECK(throws<IoError>([&] { load_ell(dir / "no_such_file.bin"); }));
    CHECK(throws<IoError>([&] { save(e, dir / "no_such_dir" / "x.bin"); }));
    CHECK(throws<IoError>([&] { load_ell(dir / "vt.bin"); }));  // another structure's file
    {
        auto b = good;
        b[0] = 'X';
        spit(dir / "bad_magic.bin", b);
        CHECK(throws<IoError>([&] { load_pattern(dir / "bad_magic.bin"); }));
        CHECK(throws<IoError>([&] { file_kind(dir / "bad_magic.bin"); }));
        b = good;
        b[8] = 2;  // version 2
        spit(dir / "bad_version.bin", b);
        CHECK(throws<IoError>([&] { load_pattern(dir / "bad_version.bin"); }));
        b = good;
        b[12] = 9;  // kind 9
        spit(dir / "bad_kind.bin", b);
        CHECK(throws<IoError>([&] { file_kind(dir / "bad_kind.bin"); }));
        for (const std::size_t cut : {std::size_t(0), std::size_t(7), std::size_t(15), std::size_t(20), good.size() / 2, good.size() - 1}) {
            spit(dir / "truncated.bin", std::vector<char>(good.begin(), good.begin() + (std::ptrdiff_t)cut));
            CHECK(throws<IoError>([&] { load_pattern(dir / "truncated.bin"); }));
        }
        b = good;
        b.push_back(0);
        spit(dir / "trailing.bin", b);
        CHECK(throws<IoError>([&] { load_pattern(dir / "trailing.bin"); }));
        b = good;  // a length prefix far beyond the file: must be refused before any allocation
        std::memset(b.data() + 20, 0x7f, 8);
        spit(dir / "huge_len.bin", b);
        CHECK(throws<IoError>([&] { load_pattern(dir / "huge_len.bin"); }));
        b = good;  // last per-row end changed: disagrees with the pattern table
        b[b.size() - 4] ^= 1;
        spit(dir / "bad_row_ends.bin", b);
        CHECK(throws<IntegrityError>([&] { load_pattern(dir / "bad_row_ends.bin"); }));
        auto eb = slurp(dir / "ell.bin");  // n * width no longer matches the arrays
        eb[16] ^= 1;
        spit(dir / "bad_ell_n.bin", eb);
        CHECK(throws<IoError>([&] { load_ell(dir / "bad_ell_n.bin"); }));
    }
    std::printf("%d checks, %d failed\n", checks, failed);
    return failed ? 1 : 0;
}
