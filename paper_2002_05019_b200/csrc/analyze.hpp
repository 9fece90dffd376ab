// Host-side symbolic phase of dd_aux_analyze ("very fast symbolic
// factorization step ... clique graph").  Integer work only.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ddaux {

struct Graph {  // undirected block graph (no self loops), vertex weights = interface sizes
  int n = 0;
  std::vector<std::vector<int>> adj;
  std::vector<int64_t> w;
};

struct Symbolic {
  int nblk = 0;
  std::vector<int> order;                 // order[t] = original block id at position t
  std::vector<int> pos;                   // pos[block] = t
  std::vector<std::vector<int>> st;       // st[t] = struct(t) as positions, ascending
  std::vector<int> parent;                // parent[t] position, -1 root
  std::vector<int> level;                 // level[t] = height (leaves 0)
  int nlevels = 0;
  std::vector<std::vector<int>> level_nodes;  // positions per level, ascending
  int64_t nnz_struct = 0;                 // sum |struct|
  double flops_factor = 0, flops_solve = 0;  // real-arithmetic counts (mu = 1)
};

// Builds the graph from a validated lower block-CSC pattern.
Graph graph_from_pattern(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx);

// Validates pattern; returns "" if ok, else the violated rule.
std::string validate_pattern(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx);

// Elimination game (clique completion) for a given order.
Symbolic symbolic_from_order(const Graph& g, const std::vector<int>& order);

// Algorithmic factor flops of an order (real, mu = 1), without building the full Symbolic.
double order_flops(const Graph& g, const std::vector<int>& order);

// Weighted minimum degree: degree = sum of neighbour sizes, ties to the lowest id.
std::vector<int> order_mindeg(const Graph& g);

// Nested dissection by recursive vertex separators (no METIS): BFS level structures from
// several roots + vertex-FM refinement; best of a few parameter variants by flop count.
std::vector<int> order_nd(const Graph& g);

}  // namespace ddaux
