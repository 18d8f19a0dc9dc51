// JSONL ingest behind the C ABI (po_load_jsonl): prefixopt::load_jsonl
// (reference table.hpp:225-269) on the host. It is the step before the
// reorder path, not on it, and its result is defined by
// nlohmann::json's parser and serializer (the reference's dependency,
// v3.11.3, the same header): every line is parsed as an ordered object, the
// schema is the union of keys in first-seen order, absent keys become "",
// strings are kept verbatim, null becomes "" and any other value keeps its
// compact JSON text (dump()). Blank lines (after dropping one trailing '\r')
// are skipped. Errors: a line that does not parse or is not an object ->
// PO_ERR_STRUCTURAL "jsonl: line N..."; an empty key -> PO_ERR_SCHEMA (the
// Table constructor's check). The result is handed over as one row-major
// arena + offsets, like po_load_csv. The FD config document of the same
// header family (fd.hpp:143-170) is parsed here too (po_load_fd_config).

#include <json.hpp>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/prefixopt_cuda.h"

namespace po {
void set_last_error(const std::string& msg);
}

struct po_jsonl {
  uint64_t rows = 0;
  std::vector<std::string> names;
  std::string arena;               // row-major cell bytes
  std::vector<uint64_t> offsets;   // rows * fields + 1
};

namespace {

struct Failure {
  int code;
  std::string msg;
};

// One parsed line: (field position, text) pairs in the line's key order.
using SparseRow = std::vector<std::pair<uint32_t, std::string>>;

void parse_lines(std::string_view text, std::vector<std::string>& names,
                 std::vector<SparseRow>& rows) {
  std::unordered_map<std::string, uint32_t> pos_of;
  uint64_t line_no = 0;
  size_t at = 0;
  while (at < text.size()) {  // std::getline semantics: a final line without '\n' counts
    size_t nl = text.find('\n', at);
    const size_t end = nl == std::string_view::npos ? text.size() : nl;
    std::string_view line = text.substr(at, end - at);
    at = nl == std::string_view::npos ? text.size() : nl + 1;
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    if (line.empty()) continue;
    nlohmann::ordered_json obj;
    try {
      obj = nlohmann::ordered_json::parse(line.begin(), line.end());
    } catch (const nlohmann::json::parse_error& e) {
      throw Failure{PO_ERR_STRUCTURAL, "jsonl: line " + std::to_string(line_no) + ": " + e.what()};
    }
    if (!obj.is_object())
      throw Failure{PO_ERR_STRUCTURAL, "jsonl: line " + std::to_string(line_no) + " is not an object"};
    SparseRow row;
    row.reserve(obj.size());
    for (auto it = obj.begin(); it != obj.end(); ++it) {
      auto ins = pos_of.try_emplace(it.key(), uint32_t(names.size()));
      if (ins.second) names.push_back(it.key());
      const auto& v = it.value();
      row.emplace_back(ins.first->second,
                       v.is_string() ? v.get<std::string>() : (v.is_null() ? std::string() : v.dump()));
    }
    rows.push_back(std::move(row));
  }
}

}  // namespace

extern "C" {

int po_load_jsonl(const uint8_t* data, uint64_t len, po_jsonl** out) {
  try {
    if (!out || (len && !data)) throw Failure{PO_ERR_INVALID_ARG, "null argument"};
    auto j = std::make_unique<po_jsonl>();
    std::vector<SparseRow> sparse;
    parse_lines(std::string_view(reinterpret_cast<const char*>(data), len), j->names, sparse);
    for (size_t f = 0; f < j->names.size(); ++f)  // Table's constructor check
      if (j->names[f].empty())
        throw Failure{PO_ERR_SCHEMA, "field " + std::to_string(f) + " has an empty name"};
    const size_t m = j->names.size();
    j->rows = sparse.size();
    j->offsets.assign(j->rows * m + 1, 0);
    // dense row-major arena: each sparse row scattered into its m slots
    std::vector<const std::string*> slot(m);
    uint64_t bytes = 0;
    for (const auto& r : sparse)
      for (const auto& c : r) bytes += c.second.size();
    j->arena.reserve(bytes);
    for (uint64_t r = 0; r < j->rows; ++r) {
      std::fill(slot.begin(), slot.end(), nullptr);
      for (const auto& c : sparse[r]) slot[c.first] = &c.second;
      for (size_t f = 0; f < m; ++f) {
        if (slot[f]) j->arena += *slot[f];
        j->offsets[r * m + f + 1] = j->arena.size();
      }
    }
    *out = j.release();
    return PO_OK;
  } catch (const Failure& f) {
    po::set_last_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    po::set_last_error(std::string("jsonl: ") + e.what());
    return PO_ERR_ERROR;
  }
}

int po_jsonl_info(const po_jsonl* j, uint64_t* out_rows, uint32_t* out_fields,
                  uint64_t* out_arena_bytes, uint64_t* out_names_bytes) {
  if (!j) {
    po::set_last_error("null handle");
    return PO_ERR_INVALID_ARG;
  }
  uint64_t nb = 0;
  for (const auto& n : j->names) nb += n.size();
  if (out_rows) *out_rows = j->rows;
  if (out_fields) *out_fields = uint32_t(j->names.size());
  if (out_arena_bytes) *out_arena_bytes = j->arena.size();
  if (out_names_bytes) *out_names_bytes = nb;
  return PO_OK;
}

int po_jsonl_copy(const po_jsonl* j, uint8_t* out_arena, uint64_t* out_offsets, uint8_t* out_names,
                  uint64_t* out_name_offsets) {
  if (!j || !out_offsets || !out_name_offsets) {
    po::set_last_error("null argument");
    return PO_ERR_INVALID_ARG;
  }
  if (!j->arena.empty()) std::memcpy(out_arena, j->arena.data(), j->arena.size());
  std::memcpy(out_offsets, j->offsets.data(), j->offsets.size() * sizeof(uint64_t));
  uint64_t at = 0;
  out_name_offsets[0] = 0;
  for (size_t f = 0; f < j->names.size(); ++f) {
    if (!j->names[f].empty()) std::memcpy(out_names + at, j->names[f].data(), j->names[f].size());
    at += j->names[f].size();
    out_name_offsets[f + 1] = at;
  }
  return PO_OK;
}

void po_jsonl_free(po_jsonl* j) { delete j; }

// load_fd_config (reference fd.hpp:143-164): {"groups": [["field", ...], ...]}.
// Sizes first (out arrays NULL), then the groups as CSR over names.
int po_load_fd_config(const uint8_t* data, uint64_t len, uint32_t* out_groups,
                      uint64_t* out_names, uint64_t* out_names_bytes, uint64_t* out_group_offsets,
                      uint64_t* out_name_offsets, uint8_t* out_bytes) {
  try {
    if (!out_groups || !out_names || !out_names_bytes || (len && !data))
      throw Failure{PO_ERR_INVALID_ARG, "null argument"};
    nlohmann::json doc;
    try {
      doc = nlohmann::json::parse(data, data + len);
    } catch (const nlohmann::json::parse_error& e) {
      throw Failure{PO_ERR_STRUCTURAL, std::string("fd config: ") + e.what()};
    }
    if (!doc.is_object() || !doc.contains("groups") || !doc["groups"].is_array())
      throw Failure{PO_ERR_SCHEMA, "fd config: expected an object with a \"groups\" array"};
    std::vector<std::vector<std::string>> groups;
    for (const auto& g : doc["groups"]) {
      if (!g.is_array()) throw Failure{PO_ERR_SCHEMA, "fd config: each group must be an array"};
      groups.emplace_back();
      for (const auto& nm : g) {
        if (!nm.is_string()) throw Failure{PO_ERR_SCHEMA, "fd config: field names must be strings"};
        groups.back().push_back(nm.get<std::string>());
      }
    }
    uint64_t names = 0, bytes = 0;
    for (const auto& g : groups)
      for (const auto& nm : g) {
        ++names;
        bytes += nm.size();
      }
    *out_groups = uint32_t(groups.size());
    *out_names = names;
    *out_names_bytes = bytes;
    if (out_group_offsets && out_name_offsets) {
      uint64_t k = 0, at = 0;
      out_group_offsets[0] = 0;
      out_name_offsets[0] = 0;
      for (size_t g = 0; g < groups.size(); ++g) {
        for (const auto& nm : groups[g]) {
          if (!nm.empty() && out_bytes) std::memcpy(out_bytes + at, nm.data(), nm.size());
          at += nm.size();
          out_name_offsets[++k] = at;
        }
        out_group_offsets[g + 1] = k;
      }
    }
    return PO_OK;
  } catch (const Failure& f) {
    po::set_last_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    po::set_last_error(std::string("fd config: ") + e.what());
    return PO_ERR_ERROR;
  }
}

}  // extern "C"
