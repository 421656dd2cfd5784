// ref_driver.cpp — drives the REFERENCE's own runtime (header-only C++20 under
// /root/reference/proj/include, compiled where it lies by oracle/Makefile into oracle/_ref/).
// TEST INFRASTRUCTURE: the checker for the batcher and the drop-in boundary.
//
//   vortex_ref_driver batcher <arrivals.txt> <cap> <b:ms,b:ms,...>
//       One-stage pipeline ("D" / modelD, stage max_batch = cap) on the reference
//       SimExecutor with the given profile knots.  Registers a recording ComponentFn and
//       prints, per query (input order): "<index> <batch> <dispatch_us> <complete_us>",
//       times relative to the first instant after the warm model load.
//       (runtime.hpp:617-672, executor.hpp:172-182, profile.hpp:90-109)
//
//   vortex_ref_driver replicas <arrivals.txt> <cap> <b:ms,...> <R>
//       The same stage with R members (R nodes, one instance each): the reference routes
//       every query with Runtime::pick_member (power of two choices on outstanding tags,
//       runtime.hpp:522-536, RNG seed RuntimeOptions::seed = 7) and each member batches on
//       its own.  Prints per query: "<index> <instance> <dispatch_us> <complete_us>".
//
//   vortex_ref_driver draws <seed> <R> <count>
//       The candidate pairs Runtime::pick_member draws for `count` routings over R active
//       members (runtime.hpp:528-531, sim::Rng(seed).below): "<a> <b>" per line.
//
//   vortex_ref_driver arrivals <rate_qps> <count> <seed> <poisson|constant> <start_us>
//       The reference's open-loop trace (bench::arrival_times, bench.hpp:54-67) from
//       sim::Rng(seed); one time (us) per line.
//
//   vortex_ref_driver profile <csv> <model> <size_gb> <b_max> <batch_cap>
//       Loads a profile CSV with the reference's ProfileTable::from_csv_file (profile.hpp:42-61)
//       and prints "lat <b> <latency_ms(model, size, b)>" for b = 1..b_max, then
//       "peak <batch> <throughput>" for peak(model, size, batch_cap) (profile.hpp:110-123) —
//       the round trip of the B200 stage's measured rows (profiles/emit_profile.py).
//
//   vortex_ref_driver pipeline <N> <D> <k> <B> <nq> <T>
//       Two stages C -> D in the reference Runtime (pipeline.json:7's "C" feeding "D"): modelC
//       is an upstream stand-in whose ComponentFn turns query i into its VXQ1 payload (vector
//       + late-interaction tokens, the cross-attention output of PreFLMR); the runtime hands
//       those outputs to D through emit_results / trigger_put_routed / deliver_bundle
//       (runtime.hpp:674-704, 570-592); modelD is the B200 stage.  Prints per query
//       "<index> batch=<b> id:ip:ms ...", then per D batch "handoff <B> <call_us>
//       <device_stage_us>": the wall time of the modelD call and the GPU stage inside it (needs
//       a GPU).
//
//   vortex_ref_driver operator <N> <D> <k> <B> <nq> <T>
//       Registers the B200 stage (include/vortex_b200_component.hpp over
//       libvortex_b200.so) as "modelD" in the reference Runtime and pushes B synthetic
//       queries (vx_synth.h seeds 43/44) through the reference batcher with cap 4
//       (pipeline.json:7).  Prints one line per query: "<index> <id> <id> ..." (needs a GPU).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "vortex/bench.hpp"
#include "vortex/runtime.hpp"

#ifdef VX_WITH_B200
#include <array>
#include <chrono>
#include <cmath>

#include "vortex_b200_component.hpp"
#include "vx_synth.h"
#endif

using namespace vortex;

static std::vector<std::pair<int, double>> parse_knots(const std::string& s) {
  std::vector<std::pair<int, double>> out;
  for (const auto& tok : split(s, ',')) {
    auto kv = split(tok, ':');
    out.emplace_back(std::stoi(kv.at(0)), std::stod(kv.at(1)));
  }
  return out;
}

struct World {
  sim::EventLoop loop;
  kvs::HandlerRegistry handlers;
  kvs::Store store{loop, handlers};
  exec::ProfileTable prof;
  std::unique_ptr<exec::SimExecutor> ex;
  std::unique_ptr<runtime::Runtime> rt;
  std::map<std::string, std::vector<exec::Instance*>> pools;
  runtime::PipelineSpec spec;

  World(int cap, const std::vector<std::pair<int, double>>& knots, int replicas = 1) {
    for (auto [b, ms] : knots) prof.add("modelD", 24, exec::ProfileEntry{b, ms, 1000.0 * b / ms, 1});
    ex = std::make_unique<exec::SimExecutor>(loop, prof);
    rt = std::make_unique<runtime::Runtime>(loop, store, handlers, *ex);
    for (int r = 0; r < replicas; ++r) {
      int node = ex->add_node(24);
      ex->partition_node(node, exec::MIGLayout{{24}});
      pools["modelD"].push_back(&ex->instance(node, 0));
    }
    spec.name = "search";
    spec.stages = {{"D", "modelD", cap, {}, {}}};
    spec.ingress = "D";
    spec.egress = "D";
  }
};

static int run_batcher(int argc, char** argv) {
  if (argc < 5) return 2;
  std::ifstream in(argv[2]);
  std::vector<sim::micros> arr;
  for (unsigned long long t; in >> t;) arr.push_back(t);
  const int cap = std::atoi(argv[3]);
  World w(cap, parse_knots(argv[4]));
  std::vector<std::vector<int>> batches;
  w.rt->register_component("modelD", [&](const std::vector<Payload>& inputs) {
    std::vector<int> b;
    for (const auto& p : inputs) b.push_back(std::stoi(payload_str(p)));
    batches.push_back(b);
    return inputs;  // output i <-> input i
  });
  w.rt->load_pipeline(w.spec, w.pools);  // warm start: runs the model load to completion
  const sim::micros t0 = w.loop.now();
  std::map<std::uint64_t, int> qid_of;
  for (size_t i = 0; i < arr.size(); ++i)
    w.loop.at(t0 + arr[i], [&, i] {
      qid_of[w.rt->ingress_submit("search", make_payload(std::to_string(i)))] = (int)i;
    });
  w.loop.run_all();
  std::vector<int> batch_of(arr.size(), -1);
  for (size_t b = 0; b < batches.size(); ++b)
    for (int i : batches[b]) batch_of[i] = (int)b;
  for (const auto& [qid, i] : qid_of) {
    const auto& rec = w.rt->record("search", qid);
    const auto& tr = rec.stages.at("D");
    std::printf("%d %d %llu %llu\n", i, batch_of[i], (unsigned long long)(tr.dispatch - t0),
                (unsigned long long)(rec.egress_ts - t0));
  }
  return 0;
}

static int run_replicas(int argc, char** argv) {
  if (argc < 6) return 2;
  std::ifstream in(argv[2]);
  std::vector<sim::micros> arr;
  for (unsigned long long t; in >> t;) arr.push_back(t);
  const int cap = std::atoi(argv[3]);
  const int R = std::atoi(argv[5]);
  World w(cap, parse_knots(argv[4]), R);
  w.rt->register_component("modelD", [](const std::vector<Payload>& inputs) { return inputs; });
  w.rt->load_pipeline(w.spec, w.pools);
  const sim::micros t0 = w.loop.now();
  std::map<std::uint64_t, int> qid_of;
  for (size_t i = 0; i < arr.size(); ++i)
    w.loop.at(t0 + arr[i], [&, i] {
      qid_of[w.rt->ingress_submit("search", make_payload(std::to_string(i)))] = (int)i;
    });
  w.loop.run_all();
  for (const auto& [qid, i] : qid_of) {
    const auto& rec = w.rt->record("search", qid);
    const auto& tr = rec.stages.at("D");
    std::printf("%d %d %llu %llu\n", i, tr.instance, (unsigned long long)(tr.dispatch - t0),
                (unsigned long long)(rec.egress_ts - t0));
  }
  return 0;
}

static int run_profile(int argc, char** argv) {
  if (argc < 7) return 2;
  auto t = exec::ProfileTable::from_csv_file(argv[2]);
  const std::string model = argv[3];
  const double size = std::atof(argv[4]);
  const int bmax = std::atoi(argv[5]), cap = std::atoi(argv[6]);
  for (int b = 1; b <= bmax; ++b) std::printf("lat %d %.17g\n", b, t.latency_ms(model, size, b));
  const auto& pk = t.peak(model, size, cap);
  std::printf("peak %d %.9g\n", pk.batch, pk.throughput_qps);
  return 0;
}

static int run_draws(int argc, char** argv) {
  if (argc < 5) return 2;
  sim::Rng rng(std::strtoull(argv[2], nullptr, 10));
  const std::size_t R = std::strtoull(argv[3], nullptr, 10);
  const long n = std::atol(argv[4]);
  for (long i = 0; i < n; ++i) {
    std::size_t a = rng.below(R);
    std::size_t b = rng.below(R - 1);
    if (b >= a) ++b;
    std::printf("%zu %zu\n", a, b);
  }
  return 0;
}

static int run_arrivals(int argc, char** argv) {
  if (argc < 7) return 2;
  bench::Phase ph;
  ph.rate_qps = std::atof(argv[2]);
  ph.count = std::strtoull(argv[3], nullptr, 10);
  ph.arrival = argv[5];
  sim::Rng rng(std::strtoull(argv[4], nullptr, 10));
  for (auto t : bench::arrival_times(ph, std::strtoull(argv[6], nullptr, 10), rng))
    std::printf("%llu\n", (unsigned long long)t);
  return 0;
}

#ifdef VX_WITH_B200
static std::vector<float> synth_row(uint64_t seed, uint64_t row, int dim) {
  std::vector<int32_t> v(dim);
  int64_t ss = 0;
  for (int c = 0; c < dim; ++c) {
    v[c] = vx_synth_int(seed, row, c);
    ss += (int64_t)v[c] * v[c];
  }
  std::vector<float> out(dim);
  for (int c = 0; c < dim; ++c) out[c] = vx_synth_finish(v[c], ss);
  return out;
}

static int run_operator(int argc, char** argv) {
  if (argc < 8) return 2;
  const int64_t N = std::atoll(argv[2]);
  const int D = std::atoi(argv[3]), k = std::atoi(argv[4]), B = std::atoi(argv[5]);
  const int nq = std::atoi(argv[6]);
  const int64_t T = std::atoll(argv[7]);
  const int Nd = 128, td = 128;
  vx_index_desc d{};
  d.n_docs = N;
  d.dim = D;
  d.n_shards = 1;
  d.tok_per_doc = nq ? Nd : 0;
  d.tok_dim = nq ? td : 0;
  d.tok_blocks = nq ? T : 0;
  d.max_batch = 4;
  d.max_k = k;
  d.max_qtok = nq;
  vx_index* h = nullptr;
  if (vx_index_create(&d, &h) != VX_OK || vx_index_synth(h, 42) != VX_OK ||
      (nq && vx_tokens_synth(h, 45) != VX_OK)) {
    std::fprintf(stderr, "vx: %s\n", vx_last_error());
    return 3;
  }
  World w(4, {{1, 125}, {4, 400}});  // modelD profile rows, profiles.csv:17-22; cap 4
  w.rt->register_component("modelD", vortex_b200::make_search_component(h, D, k));
  w.rt->load_pipeline(w.spec, w.pools);
  std::vector<std::uint64_t> qids;
  for (int i = 0; i < B; ++i) {
    auto q = synth_row(43, i, D);
    std::vector<float> tok;
    for (int j = 0; j < nq; ++j) {
      auto r = synth_row(44, (uint64_t)i * nq + j, td);
      tok.insert(tok.end(), r.begin(), r.end());
    }
    qids.push_back(w.rt->ingress_submit(
        "search", vortex_b200::encode_query(q.data(), D, nq ? tok.data() : nullptr, nq, td)));
  }
  w.loop.run_all();
  for (int i = 0; i < B; ++i) {
    const auto& rec = w.rt->record("search", qids[i]);
    auto res = vortex_b200::decode_result(rec.outputs.at("D"));
    std::printf("%d batch=%d", i, rec.stages.at("D").batch);
    for (const auto& r : res) std::printf(" %lld:%.9g:%.9g", (long long)r.id, r.ip, r.ms);
    std::printf("\n");
  }
  vx_index_destroy(h);
  return 0;
}

static int run_pipeline(int argc, char** argv) {
  if (argc < 8) return 2;
  const int64_t N = std::atoll(argv[2]);
  const int D = std::atoi(argv[3]), k = std::atoi(argv[4]), B = std::atoi(argv[5]);
  const int nq = std::atoi(argv[6]);
  const int64_t T = std::atoll(argv[7]);
  const int Nd = 128, td = 128;
  vx_index_desc d{};
  d.n_docs = N;
  d.dim = D;
  d.n_shards = 1;
  d.tok_per_doc = Nd;
  d.tok_dim = td;
  d.tok_blocks = T;
  d.max_batch = 4;
  d.max_k = k;
  d.max_qtok = nq;
  vx_index* h = nullptr;
  if (vx_index_create(&d, &h) != VX_OK || vx_index_synth(h, 42) != VX_OK ||
      vx_tokens_synth(h, 45) != VX_OK || vx_set_option(h, VX_OPT_GRAPHS, 1) != VX_OK ||
      vx_set_option(h, VX_OPT_STAGE_EVENTS, 1) != VX_OK) {  // the device stage time below
    std::fprintf(stderr, "vx: %s\n", vx_last_error());
    return 3;
  }
  // pipeline.json's tail: C (cap 4) -> D (cap 4); profiles.csv's modelD rows for both members
  World w(4, {{1, 125}, {4, 400}});
  w.prof.add("modelC", 24, exec::ProfileEntry{1, 20.0, 50.0, 1});
  w.prof.add("modelC", 24, exec::ProfileEntry{4, 60.0, 66.7, 1});
  int nodeC = w.ex->add_node(24);
  w.ex->partition_node(nodeC, exec::MIGLayout{{24}});
  w.pools["modelC"].push_back(&w.ex->instance(nodeC, 0));
  w.spec.stages = {{"C", "modelC", 4, {}, {}}, {"D", "modelD", 4, {}, {}}};
  w.spec.edges = {{"C", "D"}};
  w.spec.ingress = "C";
  w.spec.egress = "D";
  // upstream stand-in: query index -> VXQ1 payload (vector + tokens)
  w.rt->register_component("modelC", [&](const std::vector<Payload>& inputs) {
    std::vector<Payload> out;
    for (const auto& p : inputs) {
      const int i = std::stoi(payload_str(p));
      auto q = synth_row(43, i, D);
      std::vector<float> tok;
      for (int j = 0; j < nq; ++j) {
        auto r = synth_row(44, (uint64_t)i * nq + j, td);
        tok.insert(tok.end(), r.begin(), r.end());
      }
      out.push_back(vortex_b200::encode_query(q.data(), D, tok.data(), nq, td));
    }
    return out;
  });
  auto search = vortex_b200::make_search_component(h, D, k);
  std::vector<std::array<double, 3>> handoffs;
  w.rt->register_component("modelD", [&](const std::vector<Payload>& inputs) {
    const auto t0 = std::chrono::steady_clock::now();
    auto out = search(inputs);
    const auto t1 = std::chrono::steady_clock::now();
    vx_stats st{};
    vx_get_stats(h, &st);
    handoffs.push_back({(double)inputs.size(),
                        std::chrono::duration<double, std::micro>(t1 - t0).count(),
                        (double)st.last_step_ms * 1000.0});
    return out;
  });
  w.rt->load_pipeline(w.spec, w.pools);
  std::vector<std::uint64_t> qids;
  for (int i = 0; i < B; ++i)
    qids.push_back(w.rt->ingress_submit("search", make_payload(std::to_string(i))));
  w.loop.run_all();
  for (int i = 0; i < B; ++i) {
    const auto& rec = w.rt->record("search", qids[i]);
    auto res = vortex_b200::decode_result(rec.outputs.at("D"));
    std::printf("%d batch=%d", i, rec.stages.at("D").batch);
    for (const auto& r : res) std::printf(" %lld:%.9g:%.9g", (long long)r.id, r.ip, r.ms);
    std::printf("\n");
  }
  for (const auto& hf : handoffs) std::printf("handoff %d %.1f %.1f\n", (int)hf[0], hf[1], hf[2]);
  vx_index_destroy(h);
  return 0;
}
#endif

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s batcher|operator ...\n", argv[0]);
    return 2;
  }
  std::string mode = argv[1];
  try {
    if (mode == "batcher") return run_batcher(argc, argv);
    if (mode == "replicas") return run_replicas(argc, argv);
    if (mode == "arrivals") return run_arrivals(argc, argv);
    if (mode == "profile") return run_profile(argc, argv);
    if (mode == "draws") return run_draws(argc, argv);
#ifdef VX_WITH_B200
    if (mode == "operator") return run_operator(argc, argv);
    if (mode == "pipeline") return run_pipeline(argc, argv);
#endif
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
  return 2;
}
