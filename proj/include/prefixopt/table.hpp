#pragma once
// Immutable grid of byte-string cells (reference table.hpp:24-104). Keeps the
// reference's row-of-strings interface (cell() returns const std::string&)
// and adds the boundary form the GPU path consumes: one row-major byte arena
// plus n*m+1 offsets, built once on first use and cached with the table.

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "prefixopt/errors.hpp"

namespace prefixopt {

class Table {
 public:
  Table(std::vector<std::string> field_names, std::vector<std::vector<std::string>> rows)
      : names_(std::move(field_names)), rows_(std::move(rows)) {
    for (std::size_t i = 0; i < names_.size(); ++i) {
      if (names_[i].empty()) throw schema_error("field " + std::to_string(i) + " has an empty name");
      if (!index_.emplace(names_[i], static_cast<int>(i)).second)
        throw schema_error("duplicate field name: " + names_[i]);
    }
    for (std::size_t r = 0; r < rows_.size(); ++r)
      if (rows_[r].size() != names_.size())
        throw structural_error("row " + std::to_string(r) + " has " +
                               std::to_string(rows_[r].size()) + " cells, expected " +
                               std::to_string(names_.size()));
  }

  std::size_t row_count() const { return rows_.size(); }
  std::size_t field_count() const { return names_.size(); }
  const std::vector<std::string>& field_names() const { return names_; }
  const std::string& field_name(std::size_t f) const { return names_.at(f); }

  int field_index(std::string_view name) const {
    auto it = index_.find(std::string(name));
    return it == index_.end() ? -1 : it->second;
  }
  int require_field(std::string_view name) const {
    int f = field_index(name);
    if (f < 0) throw schema_error("unknown field: " + std::string(name));
    return f;
  }

  const std::string& cell(std::size_t row, std::size_t field) const { return rows_.at(row).at(field); }
  const std::vector<std::string>& row(std::size_t r) const { return rows_.at(r); }

  // FNV-1a 64 over length-prefixed field names then cells (table.hpp:68-87).
  std::uint64_t content_hash() const {
    std::uint64_t h = 0xcbf29ce484222325ull;
    auto feed = [&h](std::string_view s) {
      const std::uint64_t n = s.size();
      for (int i = 0; i < 8; ++i) {
        h ^= static_cast<unsigned char>(n >> (8 * i));
        h *= 0x100000001b3ull;
      }
      for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
      }
    };
    for (const auto& f : names_) feed(f);
    for (const auto& r : rows_)
      for (const auto& c : r) feed(c);
    return h;
  }
  std::string content_hash_hex() const {
    static constexpr char kHex[] = "0123456789abcdef";
    std::uint64_t h = content_hash();
    std::string s(16, '0');
    for (int i = 15; i >= 0; --i, h >>= 4) s[i] = kHex[h & 15];
    return s;
  }

  // ---- boundary form (row-major arena), built lazily ----
  struct Arena {
    std::vector<std::uint8_t> bytes;
    std::vector<std::uint64_t> offsets;  // row_count*field_count + 1
  };
  const Arena& arena() const {
    std::call_once(cache_->once, [this] {
      Arena& a = cache_->arena;
      std::uint64_t total = 0;
      for (const auto& r : rows_)
        for (const auto& c : r) total += c.size();
      a.bytes.reserve(total);
      a.offsets.reserve(rows_.size() * names_.size() + 1);
      a.offsets.push_back(0);
      for (const auto& r : rows_)
        for (const auto& c : r) {
          a.bytes.insert(a.bytes.end(), c.begin(), c.end());
          a.offsets.push_back(a.bytes.size());
        }
    });
    return cache_->arena;
  }

 private:
  struct Cache {
    std::once_flag once;
    Arena arena;
  };
  std::vector<std::string> names_;
  std::vector<std::vector<std::string>> rows_;
  std::unordered_map<std::string, int> index_;
  std::shared_ptr<Cache> cache_ = std::make_shared<Cache>();
};

}  // namespace prefixopt

// ingest (load_csv / load_jsonl / load_table*) and write_csv
#include "prefixopt/detail/table_io.hpp"
