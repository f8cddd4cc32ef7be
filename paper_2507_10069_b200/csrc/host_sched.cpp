// host_sched.cpp — the scheduler's per-pass host loop in C++ (SURVEY §8f
// row 4): the sliding-window load estimator the idle-rebalancing pass reads
// on every scheduler pass (balancer.py:115-164, engine.py:964-1004), the
// idle-instance grant rule (balancer.py:67-84), best-fit reservation
// placement (partition.py:169-184) and the elastic prefill instance
// allocator (partition.py:187-290) with the cost-model terms it evaluates
// (costmodel.py:90-160).
//
// Decisions are bit-exact with the reference: every float is computed with
// the same operations in the same order as the Python (double precision,
// sequential sums from 0, CPython's float floor division for buckets).
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <deque>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/emm.h"
#include "abi_util.h"

namespace {

// CostProfile fields used here, in the order of emm.h's EMM_COST_* indices
struct Cost {
  double prefill_rate, parallel_alpha, migration_bandwidth, decode_base, decode_batch_coeff,
      decode_kv_coeff, encode_rate, decode_batch_threshold;
  explicit Cost(const double* c)
      : prefill_rate(c[0]), parallel_alpha(c[1]), migration_bandwidth(c[2]), decode_base(c[3]),
        decode_batch_coeff(c[4]), decode_kv_coeff(c[5]), encode_rate(c[6]),
        decode_batch_threshold(c[7]) {}

  double parallel_speedup(int64_t n) const {  // costmodel.py:93-97
    return 1.0 / (parallel_alpha + (1.0 - parallel_alpha) / (double)n);
  }
  double prefill_time(int64_t tokens, int64_t n) const {  // costmodel.py:109-115
    if (n < 1) throw std::runtime_error("prefill needs at least one instance");
    if (tokens <= 0) return 0.0;
    return ((double)tokens / prefill_rate) / parallel_speedup(n);
  }
  double decode_step_time(int64_t bs, int64_t n, int64_t kv) const {  // costmodel.py:117-132
    const double share = ceil((double)bs / (double)n);
    const double kv_per = (double)kv / (double)n;
    return decode_base + decode_batch_coeff * share + decode_kv_coeff * (kv_per / 1000.0);
  }
  double migration_cost(int64_t kv) const {  // costmodel.py:134-138
    return kv <= 0 ? 0.0 : (double)kv / migration_bandwidth;
  }
  double decode_degradation(int64_t bs, int64_t kv, int64_t rem, int64_t nb,
                            int64_t na) const {  // costmodel.py:140-153
    if (bs < 1) return 0.0;
    const double delta = decode_step_time(bs, na, kv) - decode_step_time(bs, nb, kv);
    return std::max(0.0, delta * (double)rem);
  }
};

// Python's builtin sum() over floats (CPython >= 3.12: the first item, then
// Neumaier-compensated adds, the compensation folded in at the end), which
// is what the reference's sum(... for ...) expressions compute.
// Older CPython (3.10 / 3.11) adds plainly from left to right; the binding
// selects which one the running interpreter uses (emm_sched_set_float_sum).
static bool g_compensated_sum = true;

struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  void add(double x) {
    if (!any) {  // 0 (int start) + x
      f = 0.0 + x;
      any = true;
      return;
    }
    if (!g_compensated_sum) {
      f += x;
      return;
    }
    const double t = f + x;
    if (fabs(f) >= fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double value() const { return (c != 0.0 && isfinite(c)) ? f + c : f; }
};

struct Pool {  // DecodeBatchView (partition.py:62-69)
  const int64_t* output_lens;
  int64_t n_out, remaining_output, resident_kv, n_instances;
};

// partition.py:83-90
double gain_prefill(const Cost& p, int64_t batch_tokens, const std::vector<int64_t>& lens,
                    int64_t n) {
  if (lens.empty()) return 0.0;
  const double delta = p.prefill_time(batch_tokens, n) - p.prefill_time(batch_tokens, n + 1);
  PySum s;
  for (int64_t l : lens) s.add(delta / (double)std::max<int64_t>(1, l));
  return s.value();
}

// partition.py:93-111
double cost_prefill_preempt(const Cost& p, const Pool& b, int64_t victim_kv, double w) {
  if (b.n_instances <= 1) return INFINITY;
  const double migration = p.migration_cost(victim_kv);
  const double slowdown = p.decode_degradation(b.n_out, b.resident_kv, b.remaining_output,
                                               b.n_instances, b.n_instances - 1);
  const double per = migration + w * slowdown;
  PySum s;
  for (int64_t i = 0; i < b.n_out; ++i) s.add(per / (double)std::max<int64_t>(1, b.output_lens[i]));
  return s.value();
}

struct Spec {
  int64_t id, kv_need, input_len, prefill_tokens;
};

// partition.py:169-184: smallest sufficient slot first, ties on instance id
bool place(const std::vector<Spec>& reqs, const std::map<int64_t, int64_t>& headroom,
           std::vector<std::pair<int64_t, int64_t>>* out) {
  std::map<int64_t, int64_t> rem(headroom);
  out->clear();
  for (const Spec& s : reqs) {
    int64_t best_free = 0, best_id = 0;
    bool found = false;
    for (const auto& kv : rem) {
      if (kv.second < s.kv_need) continue;
      if (!found || kv.second < best_free || (kv.second == best_free && kv.first < best_id)) {
        best_free = kv.second;
        best_id = kv.first;
        found = true;
      }
    }
    if (!found) return false;
    out->emplace_back(s.id, best_id);
    rem[best_id] -= s.kv_need;
  }
  return true;
}

// CPython float floor division (Objects/floatobject.c float_divmod)
double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod) {
    if ((wx < 0) != (mod < 0)) div -= 1.0;
  }
  double floordiv;
  if (div) {
    floordiv = floor(div);
    if (div - floordiv > 0.5) floordiv += 1.0;
  } else {
    floordiv = copysign(0.0, vx / wx);
  }
  return floordiv;
}

// run `f`, mapping C++ exceptions to EMM_E_* codes + emm_last_error()
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::bad_alloc&) {
    emm_abi::set_error("host allocation failed");
    return EMM_E_OOM;
  } catch (const std::exception& e) {
    emm_abi::set_error(e.what());
    return EMM_E_INTERNAL;
  }
}

}  // namespace

// ------------------------------------------------------------ LoadEstimator
struct emm_estimator {
  Cost cost;
  double window, bucket;
  std::deque<std::pair<double, double>> events;  // (arrival time, service seconds)
  emm_estimator(const double* c, double w, double b) : cost(c), window(w), bucket(b) {}
  void drop_old(double now) {  // balancer.py:145-148
    const double cutoff = now - window;
    while (!events.empty() && events.front().first < cutoff) events.pop_front();
  }
};

extern "C" int emm_estimator_create(const double* cost, double window_seconds,
                                    double bucket_seconds, emm_estimator** out) {
  if (!cost || !out) {
    emm_abi::set_error("null argument");
    return EMM_E_INVALID;
  }
  return guarded([&] { *out = new emm_estimator(cost, window_seconds, bucket_seconds); });
}

extern "C" int emm_estimator_destroy(emm_estimator* e) {
  delete e;
  return 0;
}

extern "C" int emm_estimator_service_seconds(emm_estimator* e, int64_t input_tokens,
                                             int64_t image_tokens, int64_t output_tokens,
                                             double* out) {
  // balancer.py:130-138
  const Cost& p = e->cost;
  double s = (double)input_tokens / p.prefill_rate;
  const double per_token = p.decode_base / p.decode_batch_threshold + p.decode_batch_coeff;
  s += (double)output_tokens * per_token;
  if (image_tokens > 0) s += (double)image_tokens / p.encode_rate;
  *out = s;
  return 0;
}

extern "C" int emm_estimator_observe(emm_estimator* e, double now, int64_t input_tokens,
                                     int64_t image_tokens, int64_t output_tokens) {
  double s;
  emm_estimator_service_seconds(e, input_tokens, image_tokens, output_tokens, &s);
  return guarded([&] {
    e->events.emplace_back(now, s);
    e->drop_old(now);
  });
}

extern "C" int emm_estimator_avg_required(emm_estimator* e, double now, int64_t* out) {
  // balancer.py:150-153
  e->drop_old(now);
  PySum sum;  // sum(s for _, s in events)
  for (const auto& ev : e->events) sum.add(ev.second);
  const double work = sum.value();
  *out = std::max<int64_t>(1, (int64_t)ceil(work / e->window));
  return 0;
}

extern "C" int emm_estimator_peak_required(emm_estimator* e, double now, int64_t* out) {
  // balancer.py:155-164
  e->drop_old(now);
  if (e->events.empty()) {
    *out = 1;
    return 0;
  }
  return guarded([&] {
    std::map<int64_t, double> buckets;
    for (const auto& ev : e->events) {
      const int64_t k = (int64_t)py_floordiv(ev.first, e->bucket);
      auto it = buckets.find(k);
      if (it == buckets.end())
        buckets.emplace(k, 0.0 + ev.second);
      else
        it->second += ev.second;
    }
    double peak = -INFINITY;
    for (const auto& kv : buckets) peak = std::max(peak, kv.second);
    *out = std::max<int64_t>(1, (int64_t)ceil(peak / e->bucket));
  });
}

extern "C" int emm_estimator_required(emm_estimator* e, double now, int64_t* avg,
                                      int64_t* peak) {
  // avg_required(now) then peak_required(now), as Scheduler._rebalance_idle
  // reads them (engine.py:968-969)
  const int rc = emm_estimator_avg_required(e, now, avg);
  return rc ? rc : emm_estimator_peak_required(e, now, peak);
}

extern "C" int emm_estimator_len(emm_estimator* e, int64_t* out) {
  *out = (int64_t)e->events.size();
  return 0;
}

// ------------------------------------------------- assign_idle_instances
extern "C" int emm_assign_idle(const int64_t* group_ids, const int64_t* avg_required,
                               const int64_t* busy_counts, int64_t n_groups, int64_t n_idle,
                               int64_t* grants) {
  // balancer.py:67-84: each idle instance joins the active group with the
  // lowest burst tolerance (assigned / avg_required), ties on group id
  std::vector<int64_t> counts(busy_counts, busy_counts + n_groups);
  for (int64_t i = 0; i < n_groups; ++i) grants[i] = 0;
  std::vector<int64_t> active;
  for (int64_t i = 0; i < n_groups; ++i)
    if (avg_required[i] >= 1) active.push_back(i);
  if (active.empty()) return 0;
  for (int64_t k = 0; k < n_idle; ++k) {
    int64_t best = -1;
    double best_tol = 0.0;
    for (int64_t i : active) {
      const double tol = (double)counts[i] / (double)avg_required[i];
      if (best < 0 || tol < best_tol || (tol == best_tol && group_ids[i] < group_ids[best])) {
        best = i;
        best_tol = tol;
      }
    }
    ++counts[best];
    ++grants[best];
  }
  return 0;
}

// ------------------------------------------------------ place_reservations
extern "C" int emm_place_reservations(const int64_t* reqs, int64_t n_req,
                                      const int64_t* headroom, int64_t n_slots,
                                      int64_t* placed_instance, int32_t* ok) {
  return guarded([&] {
    std::vector<Spec> specs(n_req);
    for (int64_t i = 0; i < n_req; ++i) specs[i] = Spec{reqs[2 * i], reqs[2 * i + 1], 0, 0};
    std::map<int64_t, int64_t> h;
    for (int64_t i = 0; i < n_slots; ++i) h[headroom[2 * i]] = headroom[2 * i + 1];
    std::vector<std::pair<int64_t, int64_t>> out;
    *ok = place(specs, h, &out) ? 1 : 0;
    if (*ok)
      for (int64_t i = 0; i < n_req; ++i) placed_instance[i] = out[i].second;
  });
}

// --------------------------------------------------------- allocate_prefill
extern "C" int emm_allocate_prefill(
    const double* cost, double penalty_w, int64_t max_instances, const int64_t* reqs,
    int64_t n_req, const int64_t* idle, int64_t n_idle, const int64_t* victims, int64_t n_vic,
    const int64_t* output_lens, int64_t n_out, int64_t remaining_output, int64_t resident_kv,
    int64_t pool_instances, const int64_t* extra_homes, int64_t n_extra, int64_t* counts,
    int64_t* instance_ids, int64_t* placements, int64_t* preempted, int64_t* forced,
    int64_t* dropped, int64_t* dec_instance, int32_t* dec_forced, double* dec_gain,
    double* dec_cost) {
  return guarded([&] {
    const Cost p(cost);
    std::vector<int64_t> ids_v, pre_v, forced_v, drop_v, dinst;
    std::vector<int32_t> dforced;
    std::vector<double> dgain, dcost;
    std::vector<std::pair<int64_t, int64_t>> placed;
    bool have_placed = false;
    auto finish = [&](bool full) {
      counts[0] = full ? (int64_t)ids_v.size() : 0;
      // -1: placements is None (a later re-placement failed, partition.py:286-289)
      counts[1] = full ? (have_placed ? (int64_t)placed.size() : -1) : 0;
      counts[2] = (int64_t)pre_v.size();
      counts[3] = (int64_t)forced_v.size();
      counts[4] = (int64_t)drop_v.size();
      counts[5] = (int64_t)dinst.size();
      if (full) {
        std::vector<int64_t> s(ids_v);
        std::sort(s.begin(), s.end());
        std::copy(s.begin(), s.end(), instance_ids);
        for (size_t i = 0; have_placed && i < placed.size(); ++i) {
          placements[2 * i] = placed[i].first;
          placements[2 * i + 1] = placed[i].second;
        }
      }
      std::copy(pre_v.begin(), pre_v.end(), preempted);
      std::copy(forced_v.begin(), forced_v.end(), forced);
      std::copy(drop_v.begin(), drop_v.end(), dropped);
      for (size_t i = 0; i < dinst.size(); ++i) {
        dec_instance[i] = dinst[i];
        dec_forced[i] = dforced[i];
        dec_gain[i] = dgain[i];
        dec_cost[i] = dcost[i];
      }
    };
    if (n_req == 0) {  // partition.py:210-211: empty allocation
      counts[0] = counts[1] = counts[2] = counts[3] = counts[4] = counts[5] = 0;
      return;
    }
    const int64_t limit =
        max_instances >= 0 ? max_instances : std::max<int64_t>(1, n_idle + n_vic);
    // compute = idle by (-headroom, id)[:max(1, limit)]
    std::vector<std::pair<int64_t, int64_t>> idl(n_idle);
    for (int64_t i = 0; i < n_idle; ++i) idl[i] = {idle[2 * i], idle[2 * i + 1]};
    std::stable_sort(idl.begin(), idl.end(), [](const auto& a, const auto& b) {
      return a.second != b.second ? a.second > b.second : a.first < b.first;
    });
    const size_t take = std::min<size_t>(idl.size(), (size_t)std::max<int64_t>(1, limit));
    std::map<int64_t, int64_t> headroom;
    for (size_t i = 0; i < take; ++i) {
      ids_v.push_back(idl[i].first);
      headroom[idl[i].first] = idl[i].second;
    }
    for (int64_t i = 0; i < n_extra; ++i)
      headroom.emplace(extra_homes[2 * i], extra_homes[2 * i + 1]);  // setdefault
    struct Victim {
      int64_t id, kv_unused, kv_used, capacity;
    };
    std::vector<Victim> cand;
    for (int64_t i = 0; i < n_vic; ++i)
      if (victims[5 * i + 4])
        cand.push_back({victims[5 * i], victims[5 * i + 1], victims[5 * i + 2], victims[5 * i + 3]});
    std::stable_sort(cand.begin(), cand.end(), [](const Victim& a, const Victim& b) {
      return a.kv_unused != b.kv_unused ? a.kv_unused > b.kv_unused : a.id < b.id;
    });
    size_t ci = 0;  // candidates.pop(0) cursor
    Pool pool{output_lens, n_out, remaining_output, resident_kv, pool_instances};

    std::vector<Spec> working(n_req);
    for (int64_t i = 0; i < n_req; ++i)
      working[i] = Spec{reqs[4 * i], reqs[4 * i + 1], reqs[4 * i + 2], reqs[4 * i + 3]};
    have_placed = place(working, headroom, &placed);
    auto unsatisfied = [&]() { return !have_placed || ids_v.empty(); };

    // forced preemptions (partition.py:226-259)
    while (unsatisfied() && !working.empty()) {
      bool took = false;
      while (ci < cand.size() && (int64_t)ids_v.size() < limit) {
        if (pool.n_instances <= 1) break;
        const Victim v = cand[ci++];
        const double c = cost_prefill_preempt(p, pool, v.kv_used, penalty_w);
        headroom[v.id] = v.capacity;
        ids_v.push_back(v.id);
        pre_v.push_back(v.id);
        forced_v.push_back(v.id);
        dinst.push_back(v.id);
        dforced.push_back(1);
        dgain.push_back(NAN);
        dcost.push_back(c);
        pool.n_instances -= 1;
        took = true;
        have_placed = place(working, headroom, &placed);
        if (!unsatisfied()) break;
      }
      if (!unsatisfied()) break;
      if (ids_v.empty() && ci >= cand.size()) {
        for (const Spec& s : working) drop_v.push_back(s.id);
        working.clear();
        break;
      }
      if (!took) {
        drop_v.push_back(working.back().id);
        working.pop_back();
        have_placed = place(working, headroom, &placed);
      }
    }
    if (working.empty() || !have_placed) {  // partition.py:261-266
      for (const Spec& s : working) drop_v.push_back(s.id);
      pre_v.clear();
      forced_v.clear();
      dinst.clear();
      dforced.clear();
      dgain.clear();
      dcost.clear();
      finish(false);
      return;
    }
    // opportunistic preemptions while the modelled gain beats the cost
    // (partition.py:268-286)
    int64_t batch_tokens = 0;
    std::vector<int64_t> input_lens;
    for (const Spec& s : working) {
      batch_tokens += s.prefill_tokens;
      input_lens.push_back(s.input_len);
    }
    while (ci < cand.size() && (int64_t)ids_v.size() < limit) {
      const Victim v = cand[ci];
      if (pool.n_instances <= 1) break;
      const double g = gain_prefill(p, batch_tokens, input_lens, (int64_t)ids_v.size());
      const double c = cost_prefill_preempt(p, pool, v.kv_used, penalty_w);
      if (g <= c) break;
      ++ci;
      headroom[v.id] = v.capacity;
      ids_v.push_back(v.id);
      pre_v.push_back(v.id);
      dinst.push_back(v.id);
      dforced.push_back(0);
      dgain.push_back(g);
      dcost.push_back(c);
      pool.n_instances -= 1;
      have_placed = place(working, headroom, &placed);
    }
    finish(true);
  });
}

extern "C" int emm_sched_set_float_sum(int compensated) {
  g_compensated_sum = compensated != 0;
  return 0;
}
