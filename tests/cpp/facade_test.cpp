// The reference's engine tests (proj/tests/test_engine.cpp) written against
// the C++ façade include/econosim_b200.hpp: only the namespace differs from
// the reference's own test code. Linked against the sm_100a library (GPU) or
// the host build of the same source (CPU-only boxes).
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include "econosim_b200.hpp"

using namespace econosim_b200;

static int failures = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static EngineOptions base_options(PolicyKind kind) {  // test_engine.cpp:11-26
  EngineOptions o;
  o.policy.kind = kind;
  o.policy.tfs = 1024;
  o.policy.reserved_fraction = 0.05;
  o.policy.buffer_ratio = 0.0;
  o.cost.t_base = 0.005;
  o.cost.t_token = 1e-4;
  o.cost.sched_cost_per_exam = 0.0;
  o.predictor.model = ErrorModel::Oracle;
  o.predictor.padding_ratio = 0.0;
  o.kvc.capacity = 8192;
  o.kvc.block_size = 32;
  o.seed = 1;
  return o;
}

static Trace saturating_trace(int n, double rate, Tokens plo, Tokens phi, Tokens rlo, Tokens rhi,
                              std::uint64_t seed) {  // test_engine.cpp:28-37
  EconoLengthDist p{double(plo + phi) / 2.0, plo, phi, 0.4};
  EconoLengthDist r{double(rlo + rhi) / 2.0, rlo, rhi, 0.4};
  Trace t(static_cast<size_t>(n));
  char err[256];
  econo_generate_trace(n, rate, &p, &r, seed, reinterpret_cast<EconoTraceRecord*>(t.data()), err, sizeof(err));
  return t;
}

static long count_events(Engine& e, const std::string& kind) {
  long n = 0;
  for (const auto& ev : e.events())
    if (ev.kind == kind) ++n;
  return n;
}

int main() {
  {  // single request has the closed-form JCT (test_engine.cpp:66-80)
    EngineOptions o = base_options(PolicyKind::EconoFull);
    Trace trace = {{0.005, 100, 20}};
    Engine e(trace, o);
    MetricsReport rep = e.run();
    CHECK(rep.records.size() == 1);
    const RequestRecord& r = rep.records[0];
    const double expected = iteration_time(100, o.cost) + 20.0 * iteration_time(1, o.cost);
    CHECK(std::fabs(r.jct() - expected) <= 1e-9 * expected);
    CHECK(std::fabs(r.waiting_time) <= 1e-12);
    CHECK(r.preemption_time == 0.0);
    CHECK(rep.preemptions == 0);
  }
  {  // empty batch advances the clock by idle ticks (test_engine.cpp:99-108)
    Trace trace = {{1.0, 10, 5}};
    Engine e(trace, base_options(PolicyKind::EconoFull));
    e.step();
    CHECK(e.samples().size() == 1);
    CHECK(e.samples()[0].idle_repeat > 0);
    CHECK(e.clock() >= 1.0);
    CHECK(std::fabs(e.clock() - e.samples()[0].dt) <= 1e-12);
  }
  {  // runs are deterministic per seed (test_engine.cpp:110-125)
    Trace trace = saturating_trace(300, 40.0, 8, 64, 8, 96, 3);
    EngineOptions o = base_options(PolicyKind::EconoFull);
    o.predictor.model = ErrorModel::Lognormal;
    o.predictor.sigma = 0.3;
    o.predictor.padding_ratio = 0.10;
    Engine a(trace, o), b(trace, o);
    MetricsReport ra = a.run(), rb = b.run();
    CHECK(ra.mean_jct == rb.mean_jct);
    CHECK(a.events() == b.events());
  }
  {  // token conservation and clock identity (test_engine.cpp:127-145)
    Trace trace = saturating_trace(200, 30.0, 8, 80, 8, 64, 11);
    EngineOptions o = base_options(PolicyKind::EconoFull);
    o.predictor.model = ErrorModel::Lognormal;
    o.predictor.sigma = 0.25;
    o.predictor.padding_ratio = 0.10;
    Engine e(trace, o);
    e.run();
    CHECK(std::fabs(e.clock() - e.clock_from_samples()) <= 1e-12 * e.clock());
  }
  {  // underprediction draws the reserve first, then preempts (test_engine.cpp:181-206)
    Trace trace = saturating_trace(200, 40.0, 8, 40, 16, 120, 31);
    EngineOptions o = base_options(PolicyKind::EconoSD);
    o.predictor.model = ErrorModel::Lognormal;
    o.predictor.sigma = 0.6;
    o.policy.reserved_fraction = 0.30;
    Engine rich(trace, o);
    CHECK(rich.run().reserve_draws > 0);
    o.policy.reserved_fraction = 0.02;
    Engine poor(trace, o);
    MetricsReport rp = poor.run();
    CHECK(rp.preemptions > 0);
    CHECK(count_events(poor, "preempt") > 0);
    bool saw_lnew = false;
    for (const auto& ev : poor.events())
      if (ev.kind == "preempt" && ev.detail.find("l_new") != std::string::npos) saw_lnew = true;
    CHECK(saw_lnew);
  }
  {  // same-RL groups complete in one iteration (test_engine.cpp:208-231)
    Trace trace = saturating_trace(400, 60.0, 8, 32, 8, 48, 41);
    Engine e(trace, base_options(PolicyKind::EconoSD));
    e.run();
    std::map<RequestId, long> completion_iter;
    for (const auto& ev : e.events())
      if (ev.kind == "complete") completion_iter[ev.id] = ev.iter;
    std::map<long, std::map<std::string, std::vector<RequestId>>> sched;
    for (const auto& ev : e.events())
      if (ev.kind == "gt_schedule") sched[ev.iter][ev.detail].push_back(ev.id);
    long checked = 0;
    for (const auto& [iter, by_rl] : sched)
      for (const auto& [rl, members] : by_rl) {
        if (members.size() < 2) continue;
        ++checked;
        for (RequestId id : members) CHECK(completion_iter.at(id) == completion_iter.at(members[0]));
      }
    CHECK(checked > 0);
  }
  {  // hosted GTs finish by their slot deadline under the oracle (test_engine.cpp:233-241)
    Trace trace = saturating_trace(500, 250.0, 8, 32, 8, 128, 43);
    Engine e(trace, base_options(PolicyKind::EconoFull));
    MetricsReport rep = e.run();
    CHECK(e.hosted_slots_created() > 0);
    CHECK(e.hosted_overruns() == 0);
    CHECK(rep.preemptions == 0);
  }
  {  // infeasible request is rejected with a named error (test_engine.cpp:284-294)
    EngineOptions o = base_options(PolicyKind::EconoFull);
    o.kvc.capacity = 1024;
    Trace trace = {{0.1, 2000, 10}};
    bool threw = false;
    try {
      Engine e(trace, o);
    } catch (const SimulationError& ex) {
      threw = std::string(ex.what()).find("request 0") != std::string::npos;
    }
    CHECK(threw);
  }
  {  // config errors surface as ConfigError (policies.hpp:76-84)
    EngineOptions o = base_options(PolicyKind::EconoFull);
    o.policy.tfs = 0;
    bool threw = false;
    try {
      Engine e(Trace{{0.1, 10, 10}}, o);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // wire formats: write_trace_csv -> load_trace_csv round trip; the report as the CLI writes it
    Trace t = saturating_trace(60, 30.0, 8, 40, 8, 40, 5);
    const std::string csv = write_trace_csv(t);
    CHECK(csv.rfind("arrival_time,prompt_len,response_len\n", 0) == 0);
    const char* path = "/tmp/econosim_b200_facade_trace.csv";
    FILE* f = std::fopen(path, "w");
    std::fputs(csv.c_str(), f);
    std::fclose(f);
    Trace back = load_trace_csv(path);
    CHECK(back.size() == t.size());
    bool same = true;
    for (size_t i = 0; i < t.size(); ++i)
      same = same && back[i].arrival_time == t[i].arrival_time && back[i].prompt_len == t[i].prompt_len &&
             back[i].true_rl == t[i].true_rl;
    CHECK(same);
    MetricsReport rep = run(back, base_options(PolicyKind::EconoFull));
    const std::string js = to_json_string(rep, true, 2);
    CHECK(js.rfind("{\n  \"policy\": \"econoserve-full\",\n  \"trace_hash\": ", 0) == 0);
    CHECK(to_json_string(rep, false).find("\"records\"") == std::string::npos);
    bool threw = false;
    try {
      load_trace_csv("/nonexistent/trace.csv");
    } catch (const ConfigError& ex) {
      threw = std::string(ex.what()).find("cannot open trace file") != std::string::npos;
    }
    CHECK(threw);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "all facade checks passed", failures);
  return failures ? 1 : 0;
}
