// spmvcomp command-line harness (SPEC.md:425-500 [MODULE] bench_cli) on the device path.
//   spmvcomp_cli generate  --grid NX NY NZ [--out m.bin] [--mm m.mtx]
//   spmvcomp_cli bench     (--grid NX NY NZ | --matrix m.bin) --format ell|vt|pattern|pattern-values [--reps R] [--out json|csv]
//                          [--seed S] [--save format.bin] [--bandwidth GB/s | --machine spec.json]
//   spmvcomp_cli solve     (--grid NX NY NZ | --matrix m.bin) [--backend ell|vt|pattern] [--tol T] [--max-iter K]
//                          [--precond none|symgs|symgs:SWEEPS]
//   spmvcomp_cli model     (--bandwidth GB/s | --machine spec.json) [--formats ell,vt,pattern,pattern-values] [--out csv|json]
//   spmvcomp_cli calibrate [--out spec.json]     (writes the machine-spec file that --machine reads back: SPEC.md:476-483)
// Exit codes: 0 success, 1 verification / convergence failure, 2 usage error.
// Matrix files (layout in include/spmvcomp/io.hpp): `generate --out` writes the serialized
// StencilMatrix (and `--mm` the Matrix Market export), `bench` / `solve` take it with --matrix; --grid runs the
// generator on the device instead and touches no file.  `bench --save` writes the serialized format that was timed.
// A file that cannot be read or written is a failure (exit 1), not a usage error.
// Verification before timing: bench prints nothing but an error when the compressed kernel's y
// differs from the ELL backend's by more than 1e-12 relative per row (scale = sum |a_ik x_k|).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "spmvcomp/io.hpp"
#include "spmvcomp/spmvcomp.hpp"
#include "spmvcomp_b200.h"
#include "spmvcomp_b200/device.hpp"

namespace {

struct Usage {
    std::string msg;
};
struct Failure {
    std::string msg;
};

void ck(int rc, const char *what) {
    if (rc != SPMVB_OK) throw Failure{std::string(what) + ": " + spmvb_last_error()};
}

struct Args {
    int nx = 0, ny = 0, nz = 0, reps = 100, max_iter = 500;
    bool have_grid = false;
    std::string format = "pattern-values", backend = "pattern", out = "json", formats = "ell,vt,pattern,pattern-values";
    std::string matrix, mm, save, precond = "none", machine;
    bool out_given = false;
    double tol = 1e-8, bandwidth = 0.0;
    unsigned long long seed = 7;
};

Args parse(int argc, char **argv) {
    Args a;
    for (int i = 2; i < argc; i++) {
        const std::string k = argv[i];
        auto need = [&](int n) {
            if (i + n >= argc) throw Usage{"missing value for " + k};
        };
        if (k == "--grid") {
            need(3);
            a.nx = std::atoi(argv[i + 1]), a.ny = std::atoi(argv[i + 2]), a.nz = std::atoi(argv[i + 3]);
            a.have_grid = true;
            i += 3;
        } else if (k == "--format") { need(1); a.format = argv[++i];
        } else if (k == "--backend") { need(1); a.backend = argv[++i];
        } else if (k == "--reps") { need(1); a.reps = std::atoi(argv[++i]);
        } else if (k == "--out") { need(1); a.out = argv[++i]; a.out_given = true;
        } else if (k == "--matrix") { need(1); a.matrix = argv[++i];
        } else if (k == "--mm") { need(1); a.mm = argv[++i];
        } else if (k == "--save") { need(1); a.save = argv[++i];
        } else if (k == "--precond") { need(1); a.precond = argv[++i];
        } else if (k == "--seed") { need(1); a.seed = std::strtoull(argv[++i], nullptr, 10);
        } else if (k == "--tol") { need(1); a.tol = std::atof(argv[++i]);
        } else if (k == "--max-iter") { need(1); a.max_iter = std::atoi(argv[++i]);
        } else if (k == "--bandwidth") { need(1); a.bandwidth = std::atof(argv[++i]);
        } else if (k == "--formats") { need(1); a.formats = argv[++i];
        } else if (k == "--machine") { need(1); a.machine = argv[++i];
        } else throw Usage{"unknown option " + k};
    }
    return a;
}

spmvcomp::GridSpec grid_of(const Args &a) {
    if (!a.have_grid) throw Usage{"--grid NX NY NZ is required"};
    spmvcomp::GridSpec g{a.nx, a.ny, a.nz};
    spmvcomp::validate(g);  // std::invalid_argument on dims < 1 or more than 2^31-1 rows (grid.hpp:35-47)
    return g;
}

// A report goes to stdout and, when SPMVCOMP_REPORT_DIR is set, also into that directory as `name` (SPEC.md:500
// "env var to override report directory"; the reference does not name the variable -- this name is this repository's).
void emit(const std::string &name, const std::string &text) {
    std::fputs(text.c_str(), stdout);
    if (const char *dir = std::getenv("SPMVCOMP_REPORT_DIR"); dir && *dir) {
        const std::filesystem::path path = std::filesystem::path(dir) / name;
        std::FILE *f = std::fopen(path.string().c_str(), "w");
        if (!f || std::fputs(text.c_str(), f) < 0 || std::fclose(f) != 0) throw Failure{"cannot write the report to " + path.string()};
    }
}
template <class... A>
std::string fmt_str(const char *f, A... a) {
    const int len = std::snprintf(nullptr, 0, f, a...);
    std::string out((size_t)len + 1, '\0');
    std::snprintf(out.data(), out.size(), f, a...);
    out.resize((size_t)len);
    return out;
}

struct Handle {  // device handle with scope-bound lifetime
    spmvb_matrix *h = nullptr;
    Handle() = default;
    Handle(const Handle &) = delete;
    ~Handle() { if (h) spmvb_matrix_destroy(h); }
};
struct DVec {
    double *p = nullptr;
    explicit DVec(int64_t n) { ck(spmvb_vec_alloc(n, &p), "vec_alloc"); }
    DVec(const DVec &) = delete;
    ~DVec() { if (p) spmvb_vec_free(p); }
};

// The matrix of a run: generated on the device from --grid, or read from --matrix (then also kept on the host).
struct Source {
    spmvcomp::GridSpec grid{0, 0, 0};
    spmvcomp::StencilMatrix host;  // --matrix only
    bool from_file = false;
};

void generate_csr(const spmvcomp::GridSpec &g, Handle &csr);

Source open_matrix(const Args &a, Handle &csr) {
    Source s;
    if (a.have_grid == !a.matrix.empty()) throw Usage{"exactly one of --grid NX NY NZ and --matrix FILE is required"};
    if (a.have_grid) {
        s.grid = grid_of(a);
        generate_csr(s.grid, csr);
        return s;
    }
    s.host = spmvcomp::load_stencil(a.matrix);  // IoError -> exit 1
    s.grid = s.host.grid;
    s.from_file = true;
    ck(spmvb_csr_upload(s.host.n, s.host.n, 0, s.host.row_start.data(), s.host.cols.data(), s.host.vals.data(), &csr.h), "csr_upload");
    return s;
}

void generate_csr(const spmvcomp::GridSpec &g, Handle &csr) {
    spmvb_grid sg{};
    sg.nx = g.nx, sg.ny = g.ny, sg.nz = g.nz, sg.diagonal = 26.0, sg.off_diagonal = -1.0;
    ck(spmvb_generate_csr(&sg, 0, g.rows(), nullptr, &csr.h), "generate");
}

void build_format(const Handle &csr, const std::string &fmt, Handle &out) {
    spmvb_compress_options o{};
    o.value_table_limit = 256, o.min_pattern_rows = 1;
    if (fmt == "ell") ck(spmvb_csr_to_ell(csr.h, 0, nullptr, &out.h), "to_ell");
    else if (fmt == "vt") ck(spmvb_csr_compress_values(csr.h, &o, 0, nullptr, &out.h), "compress_values");
    else if (fmt == "pattern" || fmt == "pattern-values") {
        o.values_in_pattern = fmt == "pattern-values";
        ck(spmvb_csr_compress_patterns(csr.h, &o, nullptr, &out.h), "compress_patterns");
    } else throw Usage{"unknown format " + fmt};
}

double sync_read(const double *dev) {  // a synchronous one-element download: waits for everything queued before it
    double v = 0.0;
    ck(spmvb_vec_download(&v, dev, 1, nullptr), "vec_download");
    return v;
}

// matrix bytes per row as the byte model counts them (perf_model.hpp:49-57): what `effective_bandwidth` is quoted on
double model_bytes_per_row(const std::string &fmt, const spmvb_matrix_info &inf) {
    if (fmt == "ell") return 12.0 * inf.width;
    if (fmt == "vt") return 4.0 * (inf.width + inf.m);
    if (fmt == "pattern") return 4.0 + 4.0 * inf.m;
    return 4.0;
}

int cmd_generate(const Args &a) {
    const spmvcomp::GridSpec g = grid_of(a);
    const long long nnz = (3LL * g.nx - 2) * (3LL * g.ny - 2) * (3LL * g.nz - 2);
    long long file_bytes = 0;
    if (a.out_given || !a.mm.empty()) {  // the device generator's matrix, brought to the host and written out
        const spmvcomp::StencilMatrix m = spmvcomp::generate_matrix(g);
        if (a.out_given) {
            spmvcomp::save(m, a.out);
            file_bytes = (long long)spmvcomp::serialized_size(m);
        }
        if (!a.mm.empty()) spmvcomp::write_matrix_market(m, a.mm);
    }
    std::printf("{\"grid\": [%d, %d, %d], \"rows\": %lld, \"nnz\": %lld, \"csr_bytes\": %lld, \"file_bytes\": %lld}\n", g.nx, g.ny, g.nz,
                (long long)g.rows(), nnz, 8LL * (g.rows() + 1) + 12LL * nnz, file_bytes);
    return 0;
}

int cmd_bench(const Args &a) {
    if (a.reps < 1) throw Usage{"--reps must be >= 1"};
    if (a.out != "json" && a.out != "csv") throw Usage{"--out must be json or csv"};
    if (a.format != "ell" && a.format != "vt" && a.format != "pattern" && a.format != "pattern-values")
        throw Usage{"unknown format " + a.format};
    Handle csr, ell, fmt;
    const Source src = open_matrix(a, csr);
    const spmvcomp::GridSpec g = src.grid;
    spmvb_matrix_info cinf{};
    ck(spmvb_matrix_get_info(csr.h, &cinf), "info");
    const int64_t n = cinf.n;
    build_format(csr, "ell", ell);
    const bool is_ell = a.format == "ell";
    if (!is_ell) build_format(csr, a.format, fmt);
    const spmvb_matrix *run = is_ell ? ell.h : fmt.h;
    spmvb_matrix_info inf{}, einf{};
    ck(spmvb_matrix_get_info(run, &inf), "info");
    ck(spmvb_matrix_get_info(ell.h, &einf), "info");
    DVec x(n), y(n), y_ell(n), scale(n);
    ck(spmvb_vec_fill(x.p, n, 2, a.seed, -1.0, 1.0, 0, nullptr), "vec_fill");  // random, U[-1,1)
    // verification gate against the ELL backend
    ck(spmvb_spmv(ell.h, x.p, 0, n, y_ell.p, 0, (int32_t)n, nullptr), "spmv ell");
    ck(spmvb_spmv(run, x.p, 0, n, y.p, 0, (int32_t)n, nullptr), "spmv");
    ck(spmvb_row_abs_scale(csr.h, x.p, 0, scale.p, nullptr), "row_abs_scale");
    double worst = 0.0;
    int64_t differing = 0;
    ck(spmvb_compare(y.p, y_ell.p, scale.p, n, &worst, &differing, nullptr), "compare");
    double checksum = 0.0, checksum_ell = 0.0;
    ck(spmvb_dot(y.p, y.p, n, &checksum, nullptr), "dot");
    ck(spmvb_dot(y_ell.p, y_ell.p, n, &checksum_ell, nullptr), "dot");
    if (!(worst <= 1e-12) || !(std::fabs(checksum - checksum_ell) <= 1e-13 * std::fabs(checksum_ell)))
        throw Failure{"verification failed: max scaled deviation from the ELL backend " + std::to_string(worst)};
    // timing: one warm-up excluded, monotonic clock around reps back-to-back launches
    ck(spmvb_spmv(run, x.p, 0, n, y.p, 0, (int32_t)n, nullptr), "spmv");
    sync_read(y.p);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < a.reps; r++) ck(spmvb_spmv(run, x.p, 0, n, y.p, 0, (int32_t)n, nullptr), "spmv");
    sync_read(y.p);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double checksum_after = 0.0;
    ck(spmvb_dot(y.p, y.p, n, &checksum_after, nullptr), "dot");
    if (checksum_after != checksum) throw Failure{"verification failed: checksum changed between repetitions"};
    const double gflops = 2.0 * (double)inf.nnz * a.reps / sec / 1e9;
    const double bpr = model_bytes_per_row(a.format, inf);
    const double eff_bw = bpr * (double)n * a.reps / sec / 1e9;
    const double ratio = 12.0 * einf.width / bpr;
    long long file_bytes = 0;
    if (!a.save.empty()) {  // the serialized format (host structs through the C++ API: built on the device, copied back)
        const spmvcomp::StencilMatrix m = src.from_file ? src.host : spmvcomp::generate_matrix(g);
        if (a.format == "ell") {
            const auto f = spmvcomp::to_ell(m);
            spmvcomp::save(f, a.save), file_bytes = (long long)spmvcomp::serialized_size(f);
        } else if (a.format == "vt") {
            const auto f = spmvcomp::compress_values(m);
            spmvcomp::save(f, a.save), file_bytes = (long long)spmvcomp::serialized_size(f);
        } else {
            const auto f = spmvcomp::compress_patterns(m, a.format == "pattern-values");
            spmvcomp::save(f, a.save), file_bytes = (long long)spmvcomp::serialized_size(f);
        }
    }
    // roofline prediction for the configured MachineSpec (perf_model.hpp:59-72): --bandwidth GB/s, else the reference's default 75
    // (--machine FILE: the spec `calibrate --out FILE` wrote)
    const double mach_bw = a.bandwidth > 0.0 ? a.bandwidth : !a.machine.empty() ? spmvcomp::b200::load_machine_spec(a.machine).read_bandwidth / 1e9 : 75.0;
    const double roofline_gflops = mach_bw * (2.0 * (double)inf.nnz / (double)n) / bpr;
    const std::string stem = "bench_" + a.format + "_" + std::to_string(g.nx) + "x" + std::to_string(g.ny) + "x" + std::to_string(g.nz);
    if (a.out == "json")
        emit(stem + ".json",
             fmt_str("{\"format\": \"%s\", \"grid\": [%d, %d, %d], \"repetitions\": %d, \"wall_time\": %.9g, \"achieved_gflops\": %.6g, "
                     "\"effective_bandwidth_gbs\": %.6g, \"compression_ratio\": %.6g, \"bytes_per_row\": %.6g, \"machine_bandwidth_gbs\": %.6g, "
                     "\"roofline_gflops\": %.6g, \"checksum\": %.17g, \"checksum_ell\": %.17g, \"max_scaled_deviation_vs_ell\": %.3g, "
                     "\"rows\": %lld, \"nnz\": %lld, \"file_bytes\": %lld}\n",
                     a.format.c_str(), g.nx, g.ny, g.nz, a.reps, sec, gflops, eff_bw, ratio, bpr, mach_bw, roofline_gflops, checksum, checksum_ell, worst,
                     (long long)n, (long long)inf.nnz, file_bytes));
    else  // fixed column order
        emit(stem + ".csv",
             "format,nx,ny,nz,repetitions,wall_time,achieved_gflops,effective_bandwidth_gbs,compression_ratio,bytes_per_row,checksum\n" +
                 fmt_str("%s,%d,%d,%d,%d,%.9g,%.6g,%.6g,%.6g,%.6g,%.17g\n", a.format.c_str(), g.nx, g.ny, g.nz, a.reps, sec, gflops, eff_bw, ratio, bpr,
                         checksum));
    return 0;
}

int cmd_solve(const Args &a) {
    if (a.max_iter < 1 || !(a.tol > 0.0)) throw Usage{"--max-iter >= 1 and --tol > 0 are required"};
    if (a.backend != "ell" && a.backend != "vt" && a.backend != "pattern") throw Usage{"unknown backend " + a.backend};
    int sweeps = 0;  // SPEC.md:456 precond: none | symgs(sweeps)
    if (a.precond == "symgs") sweeps = 1;
    else if (a.precond.rfind("symgs:", 0) == 0) sweeps = std::atoi(a.precond.c_str() + 6);
    if (a.precond != "none" && sweeps < 1) throw Usage{"--precond must be none, symgs or symgs:SWEEPS with SWEEPS >= 1"};
    Handle csr, ell, fmt;
    const Source src = open_matrix(a, csr);
    const spmvcomp::GridSpec g = src.grid;
    spmvb_matrix_info cinf{};
    ck(spmvb_matrix_get_info(csr.h, &cinf), "info");
    const int64_t n = cinf.n;
    build_format(csr, "ell", ell);
    if (a.backend != "ell") build_format(csr, a.backend == "pattern" ? "pattern-values" : a.backend, fmt);
    const spmvb_matrix *run = a.backend == "ell" ? ell.h : fmt.h;
    DVec ones(n), b(n), x(n);
    ck(spmvb_vec_fill(ones.p, n, 0, 0, 0.0, 1.0, 0, nullptr), "vec_fill");
    ck(spmvb_spmv(ell.h, ones.p, 0, n, b.p, 0, (int32_t)n, nullptr), "spmv");  // b = A * ones
    std::vector<double> hist((size_t)a.max_iter + 1);
    int32_t it = 0, conv = 0;
    spmvb_grid sg{};
    sg.nx = g.nx, sg.ny = g.ny, sg.nz = g.nz;
    const int rc = sweeps > 0 ? spmvb_pcg_solve(run, csr.h, &sg, sweeps, b.p, x.p, a.max_iter, a.tol, &it, &conv, hist.data(), nullptr)
                              : spmvb_cg_solve(run, b.p, x.p, a.max_iter, a.tol, &it, &conv, hist.data(), nullptr);
    if (rc == SPMVB_ERR_DIVERGENCE) {
        std::fprintf(stderr, "divergence: %s\n", spmvb_last_error());
        return 1;
    }
    ck(rc, "cg_solve");
    spmvb_matrix_info inf{};
    ck(spmvb_matrix_get_info(run, &inf), "info");
    emit("solve_" + a.backend + "_" + std::to_string(g.nx) + "x" + std::to_string(g.ny) + "x" + std::to_string(g.nz) + ".json",
         fmt_str("{\"backend\": \"%s\", \"preconditioner\": \"%s\", \"grid\": [%d, %d, %d], \"iterations\": %d, \"converged\": %s, "
                 "\"final_residual\": %.6g, \"flops_total\": %lld}\n",
                 a.backend.c_str(), a.precond.c_str(), g.nx, g.ny, g.nz, it, conv ? "true" : "false", hist[(size_t)it],
                 (long long)it * (2LL * inf.nnz + 12LL * n) + (long long)(sweeps > 0 ? it + (conv ? 0 : 1) : 0) * sweeps * 4LL * inf.nnz));
    return conv ? 0 : 1;
}

int cmd_model(const Args &a) {
    spmvcomp::MachineSpec mach;
    if (a.bandwidth > 0.0) mach.read_bandwidth = a.bandwidth * 1e9;
    else if (!a.machine.empty()) mach = spmvcomp::b200::load_machine_spec(a.machine);
    else throw Usage{"--bandwidth GB/s (> 0) or --machine FILE is required"};
    std::vector<spmvcomp::MatrixFormat> formats;
    size_t pos = 0;
    while (pos <= a.formats.size()) {
        const size_t c = a.formats.find(',', pos);
        const std::string name = a.formats.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
        pos = c == std::string::npos ? a.formats.size() + 1 : c + 1;
        if (name.empty()) continue;
        const auto f = spmvcomp::parse_format(name);
        if (!f) throw Usage{"unknown format " + name};
        formats.push_back(*f);
    }
    // interior row of the 27-point stencil, table [-1, 26] (perf_model.hpp:82-95)
    const std::vector<spmvcomp::ModelRow> rows = spmvcomp::model_table(formats, 27, 2, mach);
    if (a.out_given && a.out == "csv") {
        emit("model.csv", spmvcomp::model_table_csv(rows));
    } else if (a.out_given && a.out == "json") {
        emit("model.json", spmvcomp::model_table_json(rows));
    } else {
        std::printf("%-16s %14s %14s %16s\n", "format", "bytes/row", "bytes/flop", "roofline Gflops");
        for (const auto &r : rows)
            std::printf("%-16s %14.6g %14.6g %16.6g\n", spmvcomp::format_name(r.format), r.cost.bytes_per_row, r.cost.bytes_per_flop,
                        r.estimate.predicted_flops / 1e9);
    }
    return 0;
}

int cmd_calibrate(const Args &a) {
    // device analogue of the STREAM-style sweep: w = 1*x + 0*y over 64 M doubles reads 16 and writes 8 bytes per element
    const int64_t n = 64LL << 20;
    DVec x(n), y(n), w(n);
    ck(spmvb_vec_fill(x.p, n, 0, 0, 0.0, 1.0, 0, nullptr), "vec_fill");
    ck(spmvb_vec_fill(y.p, n, 0, 0, 0.0, 1.0, 0, nullptr), "vec_fill");
    ck(spmvb_waxpby(1.0, x.p, 0.0, y.p, w.p, n, nullptr), "waxpby");
    sync_read(w.p);
    const int reps = 20;
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; r++) ck(spmvb_waxpby(1.0, x.p, 0.0, y.p, w.p, n, nullptr), "waxpby");
    sync_read(w.p);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double gbs = 24.0 * (double)n * reps / sec / 1e9;
    std::printf("{\"device_stream_bandwidth_gbs\": %.6g, \"kernel\": \"waxpby\", \"bytes_per_element\": 24, \"elements\": %lld}\n", gbs, (long long)n);
    if (a.out_given) {  // the machine-spec file bench's roofline column reads back with --machine
        spmvcomp::MachineSpec mach;
        mach.read_bandwidth = gbs * 1e9;
        spmvcomp::b200::save_machine_spec(mach, a.out);
        const spmvcomp::MachineSpec back = spmvcomp::b200::load_machine_spec(a.out);
        if (back.read_bandwidth != mach.read_bandwidth) throw Failure{"machine spec " + a.out + " does not round-trip"};
    }
    return 0;
}

}  // namespace

int main(int argc, char **argv) {
    try {
        if (argc < 2) throw Usage{"subcommand required: generate | bench | solve | model | calibrate"};
        const std::string cmd = argv[1];
        const Args a = parse(argc, argv);
        if (cmd == "generate") return cmd_generate(a);
        if (cmd == "bench") return cmd_bench(a);
        if (cmd == "solve") return cmd_solve(a);
        if (cmd == "model") return cmd_model(a);
        if (cmd == "calibrate") return cmd_calibrate(a);
        throw Usage{"unknown subcommand " + cmd};
    } catch (const Usage &u) {
        std::fprintf(stderr, "usage error: %s\n", u.msg.c_str());
        return 2;
    } catch (const std::invalid_argument &e) {
        std::fprintf(stderr, "invalid argument: %s\n", e.what());
        return 2;
    } catch (const Failure &f) {
        std::fprintf(stderr, "%s\n", f.msg.c_str());
        return 1;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
