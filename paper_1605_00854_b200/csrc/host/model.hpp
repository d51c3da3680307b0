// Host-side PBN model: the data the structural preprocessing consumes.
//
// Semantics follow the reference model (model.hpp:17-125) so the plans this
// library builds are byte-identical to pbn::prepare's:
//   * a predictor function is a truth table over an ordered parent list; bit v
//     of the table is the output when parents (parents[0] = least significant)
//     encode v (model.hpp:14-45);
//   * validation renormalises selection probabilities whose sum is within
//     1e-9 of 1 and rejects everything else (model.hpp:81-117).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pbn_b200 {

// Error classes; the C-ABI maps them to PBN_EMODEL / PBN_ERESOURCE
// (reference errors.hpp:10-32, exit codes pbn_main.cpp:302-311).
struct model_error : std::runtime_error {
  explicit model_error(const std::string& w) : std::runtime_error(w) {}
};
struct resource_error : std::runtime_error {
  explicit resource_error(const std::string& w) : std::runtime_error(w) {}
};

struct predictor {
  std::vector<std::uint32_t> parents;
  std::vector<std::uint64_t> bits;  // 2^|parents| output bits, packed LSB-first

  static constexpr std::uint32_t kMaxParents = 30;  // model.hpp:21

  std::uint32_t arity() const { return static_cast<std::uint32_t>(parents.size()); }
  bool output(std::uint64_t v) const { return (bits[v >> 6] >> (v & 63)) & 1u; }
  void set_output(std::uint64_t v, bool b) {
    if (b)
      bits[v >> 6] |= 1ull << (v & 63);
    else
      bits[v >> 6] &= ~(1ull << (v & 63));
  }
  static std::vector<std::uint64_t> zero_table(std::uint32_t phi) {
    return std::vector<std::uint64_t>(((1ull << phi) + 63) / 64, 0);
  }
};

struct pbn_node {
  std::string name;
  std::vector<predictor> fns;
  std::vector<double> probs;  // selection probabilities, same length as fns
  std::uint32_t nfn() const { return static_cast<std::uint32_t>(fns.size()); }
};

struct network {
  std::vector<pbn_node> nodes;
  double p = 0.0;                       // perturbation rate
  std::vector<std::uint32_t> interest;  // sorted ascending, unique

  std::uint32_t size() const { return static_cast<std::uint32_t>(nodes.size()); }
};

// model.hpp:78 tolerance on probability sums.
inline constexpr double kProbTolerance = 1e-9;

void validate_network(network& m);        // model.hpp:81-117
double network_density(const network& m);  // model.hpp:120-125

// Text format (io.hpp:16-23): "pbn <n>", "perturbation <p>", "node <name>",
// "f <prob> <table> [parents...]", optional "interest <names...>", '#' comments.
// The leftmost table character is the output for the highest valuation.
network parse_network(const std::string& text);    // io.hpp:74-197
std::string serialize_network(const network& m);   // io.hpp:205-226

// Parse failures carry the 1-based line (io.hpp parse_error).
struct parse_failure : model_error {
  parse_failure(int line, const std::string& w)
      : model_error("line " + std::to_string(line) + ": " + w) {}
};

}  // namespace pbn_b200
