#pragma once
// Drop-in for the reference's mqo/localsearch.hpp (localsearch.hpp:10-48).
#include <span>

#include "mqo/objectives.hpp"

namespace mqo {

struct TightnessTable {
  std::vector<int32_t> selected_neighbors;
};
TightnessTable build_tightness(const Graph& g, std::span<const Vertex> members);

struct GainTable {
  std::vector<int64_t> delta;
};
GainTable build_gain_table(const Graph& g, std::span<const uint8_t> side);
void apply_flip(const Graph& g, std::vector<uint8_t>& side, GainTable& gains, Vertex v);

std::vector<Vertex> greedy_maximalize(const Graph& g, std::vector<Vertex> members);
std::vector<Vertex> one_two_swap(const Graph& g, std::vector<Vertex> members);
int64_t one_flip_pass(const Graph& g, std::vector<uint8_t>& side);
int64_t two_flip_pass(const Graph& g, std::vector<uint8_t>& side);
int64_t one_two_flip(const Graph& g, std::vector<uint8_t>& side);

}  // namespace mqo
