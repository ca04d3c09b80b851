// SPDX-License-Identifier: MIT
// Problem files (problem_io.hpp:18-559 of the reference): canonical JSON text,
// parsing with validation, FNV-1a content / factor hashes.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "model.hpp"

namespace scn {
inline constexpr const char* kProblemSchema = "scenopt-problem-v1";
std::string write_problem(const Problem& p, int indent, bool factor_only);
std::string serialize_problem(const Problem& p);  // dump(2) + "\n"
Problem parse_problem(const std::string& text);   // throws Error(SCENOPT_E_PARSE_ERROR)
std::vector<std::string> validate_problem_text(const std::string& text);
uint64_t fnv1a(const std::string& bytes);
uint64_t content_hash(const Problem& p);
uint64_t factor_hash(const Problem& p);
void save_problem(const Problem& p, const std::string& path);
Problem load_problem(const std::string& path);
}  // namespace scn
