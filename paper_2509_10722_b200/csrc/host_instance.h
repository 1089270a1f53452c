// host_instance.h -- the library-owned instance behind numpmp_instance*
// (numpmp_host.h): flat stream-major incidence, shared by the generators
// (host_gen.cpp) and the problem-file reader (host_io.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

struct numpmp_instance {
  std::int64_t m = 0, n = 0;
  std::vector<double> capacities, weights;
  std::vector<std::uint8_t> kinds;
  std::vector<std::int64_t> offsets;
  std::vector<std::int32_t> routes;
  // transit instances only (TransitMetadata, transit.hpp:41-57): per stream
  // the OD index, route index and departure bin; per usable OD its stations
  std::vector<std::int32_t> t_od, t_route, t_t0, od_origin, od_dest;
  // the spatial edges (from, to) and each OD's routes as edge sequences:
  // OD q's routes are [od_route_ptr[q], od_route_ptr[q+1]), route r's edges
  // route_edges[route_ptr[r] .. route_ptr[r+1])
  std::vector<std::int32_t> edge_from, edge_to, route_edges;
  std::vector<std::int64_t> od_route_ptr, route_ptr;
  bool transit = false;
};

// Message of the last failing host call (numpmp_host_last_error), per thread.
extern thread_local std::string g_host_err;
