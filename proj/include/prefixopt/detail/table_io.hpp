#pragma once
// Table ingest and CSV output of the drop-in (reference table.hpp:106-294),
// included at the end of prefixopt/table.hpp. Same names, signatures, tables
// and exceptions as the reference:
//   load_csv     RFC-4180 text parsed on the GPU (po_load_csv, csrc/csv.cu)
//   load_jsonl   one JSON object per line (po_load_jsonl: the reference's
//                JSON library behind the C ABI, csrc/jsonl.cpp)
//   load_table / load_table_file / write_csv / TableFormat

#include <cstdint>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <string>
#include <string_view>
#include <vector>

#include "prefixopt/detail/check.hpp"
#include "prefixopt/errors.hpp"
#include "prefixopt/table.hpp"

namespace prefixopt {

enum class TableFormat { csv, jsonl };

namespace detail {

inline std::string slurp(std::istream& in) {
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

// Table from a loader handle's row-major arena + offsets and names.
template <class Info, class Copy>
Table table_from_handle(Info info, Copy copy) {
  std::uint64_t rows = 0, ab = 0, nb = 0;
  std::uint32_t fields = 0;
  check(info(&rows, &fields, &ab, &nb));
  std::string arena(ab ? ab : 1, '\0'), names(nb ? nb : 1, '\0');
  std::vector<std::uint64_t> off(rows * fields + 1), noff(fields + 1);
  check(copy(reinterpret_cast<std::uint8_t*>(arena.data()), off.data(),
             reinterpret_cast<std::uint8_t*>(names.data()), noff.data()));
  std::vector<std::string> field_names;
  field_names.reserve(fields);
  for (std::uint32_t f = 0; f < fields; ++f)
    field_names.push_back(names.substr(noff[f], noff[f + 1] - noff[f]));
  std::vector<std::vector<std::string>> grid(rows);
  for (std::uint64_t r = 0; r < rows; ++r) {
    grid[r].reserve(fields);
    for (std::uint32_t f = 0; f < fields; ++f) {
      const std::uint64_t i = r * fields + f;
      grid[r].push_back(arena.substr(off[i], off[i + 1] - off[i]));
    }
  }
  return Table(std::move(field_names), std::move(grid));
}

// A cell needs quoting when empty or holding a comma, quote, CR or LF
// (reference table.hpp:180-194); quotes are doubled inside.
inline void put_csv_cell(std::ostream& out, std::string_view cell) {
  if (!cell.empty() && cell.find_first_of(",\"\r\n") == std::string_view::npos) {
    out << cell;
    return;
  }
  out.put('"');
  std::size_t from = 0;
  for (std::size_t q; (q = cell.find('"', from)) != std::string_view::npos; from = q + 1)
    out << cell.substr(from, q + 1 - from) << '"';
  out << cell.substr(from) << '"';
}

}  // namespace detail

inline Table load_csv(std::istream& in) {
  const std::string text = detail::slurp(in);
  po_csv* h = nullptr;
  detail::check(po_load_csv(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(),
                            PO_LOC_HOST, &h, nullptr));
  struct Free {
    po_csv* h;
    ~Free() { po_csv_free(h); }
  } guard{h};
  return detail::table_from_handle(
      [&](std::uint64_t* r, std::uint32_t* f, std::uint64_t* ab, std::uint64_t* nb) {
        return po_csv_info(h, r, f, ab, nb);
      },
      [&](std::uint8_t* a, std::uint64_t* o, std::uint8_t* n, std::uint64_t* no) {
        return po_csv_copy(h, PO_LOC_HOST, a, o, n, no, nullptr);
      });
}

inline Table load_jsonl(std::istream& in) {
  const std::string text = detail::slurp(in);
  po_jsonl* h = nullptr;
  detail::check(po_load_jsonl(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(), &h));
  struct Free {
    po_jsonl* h;
    ~Free() { po_jsonl_free(h); }
  } guard{h};
  return detail::table_from_handle(
      [&](std::uint64_t* r, std::uint32_t* f, std::uint64_t* ab, std::uint64_t* nb) {
        return po_jsonl_info(h, r, f, ab, nb);
      },
      [&](std::uint8_t* a, std::uint64_t* o, std::uint8_t* n, std::uint64_t* no) {
        return po_jsonl_copy(h, a, o, n, no);
      });
}

inline Table load_table(std::istream& in, TableFormat format) {
  return format == TableFormat::jsonl ? load_jsonl(in) : load_csv(in);
}

inline Table load_table_file(const std::string& path, TableFormat format) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw io_error("cannot open table file: " + path);
  return load_table(in, format);
}

// Header line then one line per row, every line ending in '\n'.
inline void write_csv(const Table& t, std::ostream& out) {
  auto line = [&](auto&& field_at) {
    for (std::size_t f = 0; f < t.field_count(); ++f) {
      if (f) out.put(',');
      detail::put_csv_cell(out, field_at(f));
    }
    out.put('\n');
  };
  line([&](std::size_t f) -> const std::string& { return t.field_name(f); });
  for (std::size_t r = 0; r < t.row_count(); ++r)
    line([&](std::size_t f) -> const std::string& { return t.cell(r, f); });
}

}  // namespace prefixopt
