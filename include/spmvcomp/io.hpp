// Files either side of the SpMV path: binary serialization of the matrix and of the three
// formats, and the Matrix Market export the reference declares (inc/stencil.hpp:61-64).
//
// The reference states the layout in one sentence -- "little-endian, a 16-byte magic+version header, then the fields in
// declaration order with 8-byte length prefixes for variable arrays" -- and does not ship the document
// with the exact bytes, so the bytes below are this repository's choice ("parity unpinned"):
//
//   header   8 bytes  "SPMVCOMP"
//            u32      version = 1
//            u32      kind: 1 StencilMatrix, 2 EllMatrix, 3 VtCompressedMatrix, 4 PatternCompressedMatrix
//   body     the struct's fields in declaration order (inc/stencil.hpp:18-23, inc/ell.hpp:14-19,
//            inc/compress.hpp:36-41,65-70):
//            int32 / int64 / double   fixed width, little-endian
//            bool                     1 byte (0 or 1)
//            std::vector<T>           u64 element count, then the elements
//            ValueTable               its `entries` vector
//            GridSpec                 nx, ny, nz as int32
//            DisplacementPattern      `displacements` vector, `ends` vector
//   PatternCompressedMatrix with values_in_pattern == false carries, after the flag, the group ends per row as the
//   streaming kernel reads them (inc/compress.hpp:62-64): a vector<int32> of n * table.size() entries, row i holding
//   patterns[row_pattern[i]].ends.  With values_in_pattern == true the ends are in the pattern table only.
//
// Payload bytes per row of these files are what `measured_cost` reports (inc/perf_model.hpp:74-77): 324 for the ELL of
// 32^3, 116 + o(1) for vt, 12 + o(1) / 4 + o(1) for the two pattern variants; header, scalars, length prefixes and the
// value table are the "file metadata" it excludes.
//
// Errors: IoError when a file cannot be opened, read or written, has a wrong magic / version / kind, is truncated, has
// trailing bytes or array lengths that contradict its scalars; IntegrityError when the per-row ends of a pattern file
// disagree with its pattern table.  `load_*` does not run the full `validate` of inc/compress.hpp:92-95.
#pragma once
#include <cstdint>
#include <filesystem>

#include "spmvcomp/compress.hpp"
#include "spmvcomp/ell.hpp"
#include "spmvcomp/errors.hpp"
#include "spmvcomp/stencil.hpp"

namespace spmvcomp {

enum class FileKind : std::uint32_t { stencil = 1, ell = 2, vt = 3, pattern = 4 };
inline constexpr std::uint32_t kFileVersion = 1;

// Bytes `save` writes for the structure (the byte-accounting tests assert file sizes against it).
std::uint64_t serialized_size(const StencilMatrix& m);
std::uint64_t serialized_size(const EllMatrix& a);
std::uint64_t serialized_size(const VtCompressedMatrix& a);
std::uint64_t serialized_size(const PatternCompressedMatrix& a);

void save(const StencilMatrix& m, const std::filesystem::path& path);
void save(const EllMatrix& a, const std::filesystem::path& path);
void save(const VtCompressedMatrix& a, const std::filesystem::path& path);
void save(const PatternCompressedMatrix& a, const std::filesystem::path& path);

FileKind file_kind(const std::filesystem::path& path);  // reads the header only
StencilMatrix load_stencil(const std::filesystem::path& path);
EllMatrix load_ell(const std::filesystem::path& path);
VtCompressedMatrix load_vt(const std::filesystem::path& path);
PatternCompressedMatrix load_pattern(const std::filesystem::path& path);

// inc/stencil.hpp:61-64: coordinate format, 1-based indices, lower triangle only
// ("%%MatrixMarket matrix coordinate real symmetric"); std::invalid_argument when the matrix is not symmetric.
// Values are written with 17 significant digits, so reading the file back gives the same bits.
void write_matrix_market(const StencilMatrix& m, const std::filesystem::path& path);
// The reader takes "coordinate real symmetric" (mirrored) and "coordinate real general" files.
StencilMatrix read_matrix_market(const std::filesystem::path& path);

}  // namespace spmvcomp
