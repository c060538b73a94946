// Reference-side binding of hetbridge (see hetsim_bridge_hb.cpp).
#pragma once

#include <string>

#include "hetsim/bridge.hpp"
#include "hetsim/error.hpp"
#include "hetsim/grid.hpp"

namespace hetsim_hb {
std::string export_plan(const hetsim::grid::BoundaryEdge& e);
hetsim::bridge::DpRelation classify_dp_relation(const hetsim::grid::BoundaryEdge& e);
hetsim::grid::Placement placement_of_edge(const hetsim::grid::BoundaryEdge& e);
hetsim::grid::GridCoord coord_of_rank(const hetsim::grid::ModuleLayout& l, int rank);
}  // namespace hetsim_hb
