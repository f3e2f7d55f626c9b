// Nested-dissection tree over the primal (root) unknowns of the preconditioner.
//
// The reference factors the auxiliary decoupled operator with one sparse
// Cholesky over all of W^c (bddc_operator.cpp:38-50 -> sparse.cpp:74-81).  Here
// the substructure interiors and non-primal interface dofs are eliminated in
// the leaf fronts, whose Schur complements couple only the
// primal unknowns (corner dofs and one value per equality group).  With many
// substructures that coupled primal system is itself large but sparse (it
// follows the substructure lattice), so instead of one dense root it is
// factored as a multifrontal tree: the lattice is split into boxes by
// recursive halving of every axis, a primal unknown belongs to the smallest
// box that holds all of its substructures, and each box is a front
// [own unknowns | unknowns passed up] assembled from its children's Schur
// complements.  The top box is the (much smaller) dense root.
#pragma once

#include <vector>

namespace b200 {

struct CoarseLeaf {
  std::vector<int> coarse;  // primal unknown of each coarse slot of the leaf front
  int coord[3] = {0, 0, 0};  // substructure lattice position
  long long src0 = 0;        // offset of coarse slot 0 in the leaves' forward vector
};

struct CoarseTree {
  struct Front {
    int parent = -1;       // front index in the next level up (-1: the top)
    std::vector<int> own;  // primal unknowns eliminated here (ascending)
    std::vector<int> upd;  // primal unknowns passed up (ascending)
    int PE = 0, NF = 0;    // padded eliminated / total rows
    long long fv_off = 0, a_off = 0, d_off = 0, cmap_off = 0;
  };
  struct Level {  // all boxes of one depth
    std::vector<Front> fronts;
    long long arena = 0, a_size = 0, d_size = 0;
    int max_NF = 0, max_PE = 0, max_M = 0;
    // forward gather over the level's vector positions: (child, child coarse
    // slot) entries ascending by child; src = child's vector offset of the slot
    std::vector<int> ptr, child, cidx;
    std::vector<long long> src;
    // backward: position of each trailing slot in the parent's vector (the top
    // root's index for depth 1), -1 for pads; per front at cmap_off
    std::vector<int> cmap;
  };
  int depth = 0;
  std::vector<Level> levels;  // levels[0] = deepest boxes (children: the leaves), levels.back() = depth 1
  std::vector<int> top;       // primal unknowns of the top front (ascending)
  std::vector<int> top_ptr, top_child, top_cidx;  // gather CSR of the top (children: levels.back() or leaves)
  std::vector<long long> top_src;
  std::vector<std::vector<int>> leaf_cmap;  // per leaf: position of each coarse slot in levels[0]'s vector (or top index)
  std::vector<int> leaf_box;  // deepest box of each leaf
  int n_primal = 0;
  double flops = 0;       // factorization flops (fronts + top)
  double apply_bytes = 0;  // bytes read per preconditioner apply (both sweeps of every front + top)
};

/// Sharded engines: bounding box (lattice coordinates, hi exclusive) of the
/// substructures of EVERY rank that hold each primal unknown, so that all ranks
/// place an unknown in the same box; hi < 0 marks an unknown nobody holds.
struct CoarseBounds {
  std::vector<int> lo, hi;  // 3 per primal unknown
};

/// Deepest tree the lattice allows (every box of the level above can be split).
int coarse_tree_max_depth(const int lattice[3]);

/// Tree of the given depth (0 = one dense root over all primal unknowns).
/// `symbolic`: front sets, sizes and costs only (no gather or backward maps).
/// With `bounds` (a sharded engine) `leaves` are one rank's substructures: the
/// plan then holds the fronts of the boxes that rank owns and the whole top
/// front, whose contributions the ranks sum (engine.cu, root all-reduce).
CoarseTree plan_coarse_tree(const std::vector<CoarseLeaf>& leaves, const int lattice[3], int n_primal, int depth,
                            int root_inverse_max, bool symbolic = false, const CoarseBounds* bounds = nullptr);

/// Deepest tree (at most `max_depth`) whose boxes below the top each lie inside
/// one rank's block of the partition `owner` (rank per lattice cell, x fastest):
/// `max_depth` when the eight (or fewer) depth-1 boxes are rank-pure, else 0.
int coarse_tree_shard_depth(const int lattice[3], const std::vector<int>& owner, int max_depth);

/// Adds the gather and backward maps to a symbolic plan.
void complete_coarse_tree(CoarseTree& t, const std::vector<CoarseLeaf>& leaves);

/// Estimated seconds of setup + `applies` preconditioner applies for a plan.
double coarse_tree_cost(const CoarseTree& t, int applies, int root_inverse_max);

}  // namespace b200
