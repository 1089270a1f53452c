/*
 * numpmp_host.h -- host-side C-ABI of libnumpmp_cuda.so: synthetic instance
 * generation, problem validation and the reference layout, all on the host
 * (no device work).  These are the input producers of the hot path; each
 * restates one reference function so the same seed gives the bit-identical
 * Problem (checked against the reference in tests/test_host.py):
 *
 *   numpmp_gen_uncongested  gen.hpp:61-97 + rng.hpp:17-77
 *   numpmp_gen_congested    gen.hpp:103-128
 *   numpmp_degrade          gen.hpp:132-143
 *   numpmp_fail_and_prune   gen.hpp:146-223
 *   numpmp_read_problem     io.hpp:172-279 (parallel decode of NUMPB)
 *   numpmp_write_problem    io.hpp:126-170
 *   numpmp_validate         model.hpp:76-155 (+ violations_message 203-215)
 *   numpmp_build_layout     model.hpp:159-201
 */
#ifndef NUMPMP_HOST_H_
#define NUMPMP_HOST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GenSpec (gen.hpp:35-44). kind: 0 log, 1 linear, 2 mixed (GenKind);
 * weight_kind: 0 constant(weight_a), 1 uniform(weight_a, weight_b). */
typedef struct {
  int64_t m;
  int64_t n; /* 0 -> max(1, m/2) */
  double avg_links_per_stream;
  int32_t kind;
  int32_t weight_kind;
  double weight_a;
  double weight_b;
  uint64_t seed;
} numpmp_gen_spec;

/* A generated instance owned by the library (stream-major incidence). */
typedef struct numpmp_instance numpmp_instance;

/* Returns 0, or 5 (GenError) / 2 (ValidationError) with a message in
 * numpmp_host_last_error(). */
int numpmp_gen_uncongested(const numpmp_gen_spec* spec, numpmp_instance** out);
int numpmp_gen_congested(const numpmp_gen_spec* spec, double hot_link_fraction,
                         double hot_stream_fraction, numpmp_instance** out);
void numpmp_instance_sizes(const numpmp_instance* inst, int64_t* m, int64_t* n, int64_t* nnz);
/* Copies the instance out; any pointer may be null. */
void numpmp_instance_export(const numpmp_instance* inst, double* capacities, double* weights,
                            uint8_t* kinds, int64_t* stream_offsets, int32_t* route_links);
void numpmp_instance_free(numpmp_instance* inst);

/* TransitSpec (transit.hpp:22-32): time-expanded transit network, one
 * stream per (OD pair, route, departure); link id = edge * time_bins + t. */
typedef struct {
  int32_t stations;
  int32_t time_bins;
  double bin_minutes;
  int64_t spatial_edges;
  int64_t od_pairs;
  int32_t routes_per_od;
  int32_t departures_per_route;
  double seats;
  uint64_t seed;
} numpmp_transit_spec;

/* gen_transit (transit.hpp:152-287): random strongly connected spatial
 * graph, Yen k-shortest loop-free routes per OD pair, evenly spaced
 * departures; streams arriving past the horizon are dropped (count in
 * *dropped).  Returns 0 or 5 (GenError). */
int numpmp_gen_transit(const numpmp_transit_spec* spec, numpmp_instance** out, int64_t* dropped);
/* TransitMetadata of a numpmp_gen_transit instance (transit.hpp:35-57):
 * *n_ods usable OD pairs (TransitMetadata::ods, disconnected pairs skipped);
 * per stream (length n) the OD index, route index and departure bin
 * (TransitMetadata::streams); per OD its origin and destination station
 * (length *n_ods).  Any pointer may be null; size with n_ods first.
 * Returns 0, or 2 (ValidationError) for an instance not made by
 * numpmp_gen_transit. */
int numpmp_transit_meta(const numpmp_instance* inst, int64_t* n_ods, int32_t* od, int32_t* route,
                        int32_t* t0, int32_t* od_origin, int32_t* od_dest);
/* The rest of TransitMetadata: the spatial edges (from, to) and each OD's
 * routes as edge sequences (OD q: routes [od_route_ptr[q], od_route_ptr[q+1]),
 * route r: route_edges[route_ptr[r] .. route_ptr[r+1])).  Size with the
 * counts first; any pointer may be null.  Returns 0 or 2. */
int numpmp_transit_graph(const numpmp_instance* inst, int64_t* n_edges, int64_t* n_routes, int64_t* n_route_edges,
                         int32_t* edge_from, int32_t* edge_to, int64_t* od_route_ptr, int64_t* route_ptr,
                         int32_t* route_edges);
/* write_transit_metadata (io.hpp:444-467): the "NUMT 1" sidecar, the same
 * bytes as the reference.  Returns 0 or 6 (IoError). */
int numpmp_write_transit_metadata(const char* path, int32_t stations, int32_t time_bins, double bin_minutes,
                                  double seats, int64_t dropped, int64_t n_edges, const int32_t* edge_from,
                                  const int32_t* edge_to, int64_t n_ods, const int32_t* od_origin,
                                  const int32_t* od_dest, const int64_t* od_route_ptr, const int64_t* route_ptr,
                                  const int32_t* route_edges, int64_t n_streams, const int32_t* s_od,
                                  const int32_t* s_route, const int32_t* s_t0);

/* In-place capacity degradation with the reference's draw order. */
int numpmp_degrade(int64_t m, double* capacities, double p_degrade, double factor, uint64_t seed);
/* Problem files (io.hpp:126-279): read_problem of the text "NUMP 1" or the
 * binary "NUMPB 1" container (sniffed by magic) into an instance; returns 0,
 * 6 (IoError, the reference's message) or 2 (ValidationError from
 * build_problem).  write_problem: encoding 0 auto (binary when m >= 1e6),
 * 1 text, 2 binary; the same bytes as the reference writer. */
int numpmp_read_problem(const char* path, numpmp_instance** out);
/* write_trace_csv (io.hpp:393-404): "iter,r_norm,s_norm,rho,objective" and
 * one %.17g row per trace record, the same bytes as the reference.
 * Returns 0 or 6 (IoError, the reference's message). */
int numpmp_write_trace_csv(const char* path, int64_t rows, const int64_t* iter, const double* r_norm,
                           const double* s_norm, const double* rho, const double* objective);
int numpmp_write_problem(int64_t m, int64_t n, const double* capacities, const double* weights,
                         const uint8_t* kinds, const int64_t* offsets, const int32_t* routes,
                         const char* path, int encoding);
/* fail_and_prune (gen.hpp:181-223): the pruned instance plus the PruneMap
 * (gen.hpp:146-178): link_map[m] (new id or -1), stream_map[n] (new id or -1). */
int numpmp_fail_and_prune(int64_t m, int64_t n, const double* capacities, const double* weights,
                          const uint8_t* kinds, const int64_t* offsets, const int32_t* routes,
                          double p_fail, uint64_t seed, numpmp_instance** out, int32_t* link_map,
                          int64_t* stream_map);

/* Model validation; returns the number of violations and writes the
 * reference's "invalid problem: [...]" message (truncated to msg_cap). */
int64_t numpmp_validate(int64_t m, int64_t n, const double* capacities, const double* weights,
                        const uint8_t* kinds, const int64_t* stream_offsets,
                        const int32_t* route_links, char* msg, int64_t msg_cap);

/* The reference TerminalLayout on the host (terminal_link[J],
 * link_offsets[m+1], link_terminals[J], link_counts[m]). */
int numpmp_build_layout(int64_t m, int64_t n, const int64_t* stream_offsets,
                        const int32_t* route_links, int32_t* terminal_link,
                        int64_t* link_offsets, int64_t* link_terminals, int32_t* link_counts);

const char* numpmp_host_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NUMPMP_HOST_H_ */
