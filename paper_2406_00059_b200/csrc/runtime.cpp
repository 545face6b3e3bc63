// runtime.cpp -- the native host runtime above the engine (include/conveyor.h "Native host
// runtime"): the scheduler of PAPER.md:146 (Fig. 4) in C++ threads.
//
//   driver (the thread calling cvy_runtime_run): cvy_step back to back while any request is
//       decoding (continuous batching, step (2)); otherwise it sleeps on a condition variable
//       until a tool finishes or an observation is injected;
//   poller (one thread, the ring's single consumer): cvy_poll_segments while decoding
//       continues (step (8), "periodically polls"); every polled piece goes through the plan
//       callback and is dispatched at once (Partial) or held until the
//       round's FINAL (Sequential, reading R15);
//   workers (n_workers threads): execute pieces; pieces of one (request, round, instance)
//       run serially in arrival order, instances in parallel, dependencies honoured
//       (planning DAG) -- the same rules as the O-3 schedule the tests
//       recompute from these logs;
//   rounds: when a round's FINAL is in and all its pieces have executed, the observation is
//       injected (cvy_inject_observation, step (g)); an `abort` piece cancels
//       its request when it completes (validator); with max_inflight the
//       finished request's slot is released at once and the next request admitted (NEXT-3).
//
// Only the public C ABI of the engine is used.  Lock order: runtime mutex, then (inside the
// engine calls) the engine's mutex; cvy_step and cvy_poll_segments run without the runtime
// mutex held.
#include <time.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/conveyor.h"

cvy_status cvy_internal_fail(cvy_status st, const std::string& msg);  // engine.cu (thread-local last error)

namespace {

using Clock = std::chrono::steady_clock;

double thread_cpu_s() {
    timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

struct Piece {
    cvy_piece_plan plan;
    double t_avail = -1, t_disp = -1, t_begin = -1, t_end = -1;
    uint32_t token = 0;
    bool dispatched = false, done = false;
};

struct RoundState {
    double t_start = -1, t_final = -1;
    std::deque<Piece> pieces;  // deque: stable references while the poller appends
    std::vector<uint32_t> held; // Sequential: pieces waiting for FINAL
};

struct Req {
    std::vector<int32_t> prompt;
    uint32_t synth_prefix = 0;
    uint64_t synth_seed = 0;
    std::vector<std::vector<int32_t>> forced, obs;
    std::vector<int32_t> tool;
    uint32_t reserve = 0;
    double t_arrival = 0;
    // state
    uint64_t rid = 0;
    bool submitted = false, final_seen = false, done = false, released = false;
    uint32_t round = 0;
    double t_submit = -1, t_done = -1, t_abort = -1;
    std::vector<RoundState> rounds;
    int pending = 0;  // dispatched pieces not yet finished
};

struct Inst {
    bool busy = false;
    std::deque<uint32_t> q;  // piece indices waiting for this instance
};

struct Task {
    uint32_t req, round, piece;
};

}  // namespace

struct cvy_runtime {
    cvy_engine* e = nullptr;
    cvy_runtime_config cfg{};
    std::mutex mu;
    std::condition_variable cv_driver, cv_work;
    std::vector<Req> reqs;
    std::unordered_map<uint64_t, uint32_t> by_rid;
    std::deque<uint32_t> waiting;  // not yet admitted, in arrival order
    uint32_t active = 0;           // not finished
    uint32_t inflight = 0;         // admitted, not finished
    std::map<std::tuple<uint32_t, uint32_t, int32_t>, Inst> inst;
    std::deque<Task> ready;
    bool stop = false;
    Clock::time_point t0;
    std::string err;
    cvy_rt_stats st{};

    double now() const { return std::chrono::duration<double>(Clock::now() - t0).count(); }

    // ---------------------------------------------------------------- request lifecycle
    cvy_status submit(uint32_t i) {  // caller holds mu
        Req& r = reqs[i];
        cvy_request_desc d;
        std::memset(&d, 0, sizeof(d));
        d.tool_id = r.tool[0];
        d.mode = cfg.mode;
        d.prompt = r.prompt.data();
        d.prompt_len = (uint32_t)r.prompt.size();
        d.synth_prefix_len = r.synth_prefix;
        d.synth_seed = r.synth_seed;
        d.max_new_tokens = (uint32_t)r.forced[0].size();
        d.forced = r.forced[0].data();
        d.forced_len = (uint32_t)r.forced[0].size();
        d.reserve_tokens = r.reserve;
        r.t_submit = now();
        cvy_status s = cvy_submit_request(e, &d, &r.rid);
        if (s != CVY_OK) return s;
        r.submitted = true;
        inflight++;
        r.rounds.emplace_back();
        r.rounds.back().t_start = r.t_submit;
        by_rid[r.rid] = i;
        return CVY_OK;
    }

    // admit waiting requests that have arrived, in arrival order, within max_inflight; a full
    // engine (CVY_E_FULL: no free slot or pages) keeps the request at the head of the queue until
    // a finished request is released; any other error fails the run
    void admit(double t) {  // caller holds mu
        while (!waiting.empty() && reqs[waiting.front()].t_arrival <= t &&
               (cfg.max_inflight == 0 || inflight < cfg.max_inflight)) {
            const uint32_t k = waiting.front();
            cvy_status s = submit(k);
            if (s == CVY_E_FULL && inflight > 0) break;
            waiting.pop_front();
            if (s != CVY_OK) {
                err = std::string("submit: ") + cvy_last_error();
                reqs[k].done = true;
                active--;
            }
        }
    }

    void finish(uint32_t i, double t) {  // caller holds mu
        Req& r = reqs[i];
        r.done = true;
        r.t_done = t;
        active--;
        inflight--;
        if (cfg.max_inflight > 0 || !waiting.empty()) {
            // abort-and-refill (NEXT-3): the slot and its pages go back now (applied at the next
            // step boundary) and a waiting request takes them
            if (cvy_release_request(e, r.rid) == CVY_OK) r.released = true;
            admit(t);
        }
        cv_driver.notify_all();
    }

    void maybe_advance(uint32_t i, double t) {  // caller holds mu
        Req& r = reqs[i];
        if (r.done || !r.final_seen || r.pending > 0) return;
        RoundState& rs = r.rounds[r.round];
        for (const Piece& p : rs.pieces)
            if (!p.done) return;
        if (r.t_abort >= 0 || r.round + 1 >= r.forced.size()) {
            finish(i, t);
            return;
        }
        const uint32_t nxt = r.round + 1;
        const std::vector<int32_t>& ob = r.obs[r.round];
        r.round = nxt;
        r.final_seen = false;
        r.rounds.emplace_back();
        r.rounds.back().t_start = t;
        cvy_status s = cvy_inject_observation(e, r.rid, ob.data(), (uint32_t)ob.size(), (uint32_t)r.forced[nxt].size(),
                                              r.forced[nxt].data(), (uint32_t)r.forced[nxt].size());
        st.injections++;
        if (s != CVY_OK) {
            err = std::string("inject: ") + cvy_last_error();
            finish(i, t);
            return;
        }
        cv_driver.notify_all();
    }

    // ---------------------------------------------------------------- dispatch / execution
    bool deps_done(const RoundState& rs, const Piece& p) const {
        for (uint32_t d = 0; d < p.plan.n_deps; ++d) {
            const int k = p.plan.deps[d];
            if (k < 0 || k >= (int)rs.pieces.size() || !rs.pieces[(size_t)k].done) return false;
        }
        return true;
    }

    void dispatch(uint32_t i, uint32_t rnd, uint32_t j, double t) {  // caller holds mu
        Req& r = reqs[i];
        RoundState& rs = r.rounds[rnd];
        Piece& p = rs.pieces[j];
        if (p.dispatched || !deps_done(rs, p)) return;  // dependants retry when a dep finishes
        p.dispatched = true;
        p.t_disp = t;
        r.pending++;
        Inst& in = inst[std::make_tuple(i, rnd, p.plan.instance)];
        if (in.busy) {
            in.q.push_back(j);
        } else {
            in.busy = true;
            ready.push_back({i, rnd, j});
            cv_work.notify_one();
        }
    }

    void piece_done(const Task& tk, double t) {  // caller holds mu
        Req& r = reqs[tk.req];
        RoundState& rs = r.rounds[tk.round];
        Piece& p = rs.pieces[tk.piece];
        p.t_end = t;
        p.done = true;
        r.pending--;
        if (p.plan.abort && r.t_abort < 0 && !r.done) {
            r.t_abort = t;
            cvy_cancel_request(e, r.rid);
            st.cancels++;
        }
        Inst& in = inst[std::make_tuple(tk.req, tk.round, p.plan.instance)];
        if (!in.q.empty()) {
            const uint32_t nj = in.q.front();
            in.q.pop_front();
            ready.push_back({tk.req, tk.round, nj});
            cv_work.notify_one();
        } else {
            in.busy = false;
        }
        // dependants waiting for this piece
        if (!r.done)
            for (uint32_t k = 0; k < rs.pieces.size(); ++k) {
                Piece& q = rs.pieces[k];
                if (q.dispatched) continue;
                bool mine = false;
                for (uint32_t d = 0; d < q.plan.n_deps; ++d) mine = mine || q.plan.deps[d] == (int)tk.piece;
                if (mine && (cfg.mode == CVY_MODE_PARTIAL || (tk.round < r.round || r.final_seen)))
                    dispatch(tk.req, tk.round, k, std::max(t, q.t_avail));
            }
        if (tk.round == r.round) maybe_advance(tk.req, t);
    }

    void worker() {
        const double c0 = thread_cpu_s();
        std::unique_lock<std::mutex> lk(mu);
        while (true) {
            cv_work.wait(lk, [&] { return stop || !ready.empty(); });
            if (stop && ready.empty()) break;
            const Task tk = ready.front();
            ready.pop_front();
            Piece& p = reqs[tk.req].rounds[tk.round].pieces[tk.piece];
            p.t_begin = now();
            const double cost = p.plan.cost_ms;
            lk.unlock();
            // the tool stub: the caller's seeded cost model occupies this executor
            if (cost > 0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(cost));
            lk.lock();
            st.pieces++;
            piece_done(tk, now());
        }
        st.worker_cpu_s += thread_cpu_s() - c0;
    }

    void on_record(const cvy_segment& r, const uint8_t* data, double t, uint32_t i, const cvy_piece_plan* plan,
                   uint32_t j) {  // caller holds mu
        Req& q = reqs[i];
        if (q.done) return;
        const uint32_t rnd = q.round;
        RoundState& rs = q.rounds[rnd];
        const bool is_final = (r.flags & CVY_SEG_FINAL) != 0;
        (void)data;
        if (plan && !plan->skip && j == rs.pieces.size()) {
            rs.pieces.emplace_back();
            Piece& p = rs.pieces.back();
            p.plan = *plan;
            p.plan.n_deps = std::min<uint32_t>(p.plan.n_deps, 8);
            p.t_avail = t;
            p.token = r.token_index;
            if (cfg.mode == CVY_MODE_PARTIAL)
                dispatch(i, rnd, j, t);
            else
                rs.held.push_back(j);
        }
        if (is_final) {
            rs.t_final = t;
            q.final_seen = true;
            if (r.flags & CVY_SEG_CANCELLED) {
                finish(i, q.t_abort >= 0 ? q.t_abort : t);
                return;
            }
            if (cfg.mode == CVY_MODE_SEQUENTIAL) {
                for (uint32_t k : rs.held) dispatch(i, rnd, k, t);
                rs.held.clear();
            }
            for (uint32_t k = 0; k < rs.pieces.size(); ++k) dispatch(i, rnd, k, t);
            maybe_advance(i, t);
        }
    }

    void poller() {
        const double c0 = thread_cpu_s();
        std::vector<cvy_segment> recs(1024);
        std::vector<uint8_t> bytes(1 << 20);
        std::vector<cvy_piece_plan> plans(1024);
        std::vector<uint32_t> req_of(1024), idx_of(1024);
        std::vector<char> has_plan(1024);
        const unsigned sleep_us = cfg.poll_sleep_us ? cfg.poll_sleep_us : 20;
        while (true) {
            {
                std::lock_guard<std::mutex> lk(mu);
                if (stop) break;
            }
            uint32_t n = 0;
            size_t used = 0;
            cvy_status s = cvy_poll_segments(e, recs.data(), (uint32_t)recs.size(), &n, bytes.data(), bytes.size(), &used);
            if (s == CVY_E_AGAIN) {
                std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
                continue;
            }
            const double t = now();
            if (s != CVY_OK) {
                std::lock_guard<std::mutex> lk(mu);
                err = std::string("poll: ") + cvy_last_error();
                stop = true;
                cv_driver.notify_all();
                cv_work.notify_all();
                break;
            }
            const double d0 = thread_cpu_s();
            // plans first, without the runtime lock (the callback may be slow); only this thread
            // appends pieces, so the piece index of a round cannot change meanwhile
            size_t off = 0;
            std::unordered_map<uint64_t, uint32_t> next_j;  // (request, round) -> next piece index in this batch
            for (uint32_t k = 0; k < n; ++k) {
                const cvy_segment& r = recs[k];
                const uint8_t* data = bytes.data() + off;
                off += r.byte_len;
                has_plan[k] = 0;
                uint32_t i = 0, rnd = 0, j0 = 0;
                int32_t tool = -1;
                bool live = false;
                {
                    std::lock_guard<std::mutex> lk(mu);
                    auto it = by_rid.find(r.req_id);
                    if (it != by_rid.end() && !reqs[it->second].done) {
                        i = it->second;
                        rnd = reqs[i].round;
                        tool = reqs[i].tool[rnd];
                        j0 = (uint32_t)reqs[i].rounds[rnd].pieces.size();
                        live = true;
                    }
                }
                req_of[k] = live ? i : UINT32_MAX;
                if (!live) continue;
                const bool is_final = (r.flags & CVY_SEG_FINAL) != 0;
                if (tool >= 0 && (!is_final || r.byte_len > 0)) {
                    const uint64_t key = ((uint64_t)i << 20) | rnd;
                    auto jt = next_j.find(key);
                    const uint32_t j = jt == next_j.end() ? j0 : jt->second;
                    std::memset(&plans[k], 0, sizeof(cvy_piece_plan));
                    cfg.plan(cfg.plan_user, i, rnd, j, data, r.byte_len, r.flags, &plans[k]);
                    has_plan[k] = 1;
                    idx_of[k] = j;
                    next_j[key] = plans[k].skip ? j : j + 1;
                }
                // a FINAL advances the round only when processed below: later records of this
                // batch belong to the next round only after an injection, which happens on the
                // runtime's own threads after this batch is handled
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                off = 0;
                for (uint32_t k = 0; k < n; ++k) {
                    const uint8_t* data = bytes.data() + off;
                    off += recs[k].byte_len;
                    if (req_of[k] == UINT32_MAX) continue;
                    on_record(recs[k], data, t, req_of[k], has_plan[k] ? &plans[k] : nullptr, idx_of[k]);
                }
                st.records += n;
                st.dispatch_cpu_s += thread_cpu_s() - d0;
            }
        }
        std::lock_guard<std::mutex> lk(mu);
        st.poller_cpu_s += thread_cpu_s() - c0;
    }
};

cvy_status cvy_runtime_create(cvy_engine* e, const cvy_runtime_config* cfg, cvy_runtime** out) {
    if (!out) return cvy_internal_fail(CVY_E_INVAL, "null out");
    *out = nullptr;
    if (!e || !cfg || !cfg->plan || cfg->n_workers < 1 || cfg->n_workers > 4096)
        return cvy_internal_fail(CVY_E_INVAL, "runtime: engine, plan callback and 1..4096 workers required");
    if (cfg->mode != CVY_MODE_PARTIAL && cfg->mode != CVY_MODE_SEQUENTIAL)
        return cvy_internal_fail(CVY_E_INVAL, "runtime: bad mode");
    cvy_runtime* rt = new cvy_runtime();
    rt->e = e;
    rt->cfg = *cfg;
    *out = rt;
    return CVY_OK;
}

cvy_status cvy_runtime_run(cvy_runtime* rt, const cvy_rt_request* reqs, uint32_t n, double timeout_s) {
    if (!rt || (!reqs && n)) return cvy_internal_fail(CVY_E_INVAL, "runtime: null argument");
    for (uint32_t i = 0; i < n; ++i) {
        const cvy_rt_request& q = reqs[i];
        if (!q.prompt || q.prompt_len < 1 || !q.rounds || q.n_rounds < 1)
            return cvy_internal_fail(CVY_E_INVAL, "runtime: request needs a prompt and >= 1 round");
        if (!(q.t_arrival >= 0)) return cvy_internal_fail(CVY_E_INVAL, "runtime: t_arrival must be >= 0");
        for (uint32_t k = 0; k < q.n_rounds; ++k)
            if (!q.rounds[k].forced || q.rounds[k].forced_len < 1 || (q.rounds[k].observation_len && !q.rounds[k].observation))
                return cvy_internal_fail(CVY_E_INVAL, "runtime: a round needs >= 1 forced token");
    }
    // copy the descriptors
    rt->reqs.assign(n, Req());
    for (uint32_t i = 0; i < n; ++i) {
        const cvy_rt_request& q = reqs[i];
        Req& r = rt->reqs[i];
        r.prompt.assign(q.prompt, q.prompt + q.prompt_len);
        r.synth_prefix = q.synth_prefix_len;
        r.synth_seed = q.synth_seed;
        r.t_arrival = q.t_arrival;
        for (uint32_t k = 0; k < q.n_rounds; ++k) {
            const cvy_round_desc& d = q.rounds[k];
            r.forced.emplace_back(d.forced, d.forced + d.forced_len);
            r.obs.emplace_back(d.observation, d.observation + d.observation_len);
            r.tool.push_back(d.tool_id);
            if (k > 0) r.reserve += d.forced_len + q.rounds[k - 1].observation_len + 2;
        }
        r.reserve += q.rounds[0].observation_len;
    }
    rt->by_rid.clear();
    rt->inst.clear();
    rt->ready.clear();
    rt->waiting.clear();
    rt->stop = false;
    rt->err.clear();
    rt->st = cvy_rt_stats{};
    rt->t0 = Clock::now();
    const double c0 = thread_cpu_s();
    cvy_status result = CVY_OK;
    {
        std::lock_guard<std::mutex> lk(rt->mu);
        rt->active = n;
        rt->inflight = 0;
        std::vector<uint32_t> order(n);
        for (uint32_t i = 0; i < n; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t a, uint32_t b) { return rt->reqs[a].t_arrival < rt->reqs[b].t_arrival; });
        for (uint32_t i : order) rt->waiting.push_back(i);
        rt->admit(0.0);
        if (!rt->err.empty()) result = CVY_E_FULL;
    }
    if (result != CVY_OK) {
        for (auto& r : rt->reqs)
            if (r.submitted) cvy_cancel_request(rt->e, r.rid);
        cvy_sync(rt->e);
        return cvy_internal_fail(result, rt->err);
    }
    std::thread poller([rt] { rt->poller(); });
    std::vector<std::thread> workers;
    for (uint32_t w = 0; w < rt->cfg.n_workers; ++w) workers.emplace_back([rt] { rt->worker(); });
    // driver: decoding iterations back to back while any request decodes
    while (true) {
        bool busy = false;
        {
            std::unique_lock<std::mutex> lk(rt->mu);
            if (rt->active == 0 || rt->stop) break;
            rt->admit(rt->now());
            for (const Req& r : rt->reqs)
                if (r.submitted && !r.done && !r.final_seen) {
                    busy = true;
                    break;
                }
            if (!busy) rt->cv_driver.wait_for(lk, std::chrono::microseconds(500));
        }
        if (busy) {
            cvy_status s = cvy_step(rt->e, nullptr);
            if (s != CVY_OK) {
                std::lock_guard<std::mutex> lk(rt->mu);
                rt->err = std::string("step: ") + cvy_last_error();
                result = CVY_E_STATE;
                break;
            }
            rt->st.steps++;
        }
        if (rt->now() > timeout_s) {
            std::lock_guard<std::mutex> lk(rt->mu);
            rt->err = "runtime: timeout";
            result = CVY_E_STATE;
            break;
        }
    }
    cvy_sync(rt->e);
    {
        std::lock_guard<std::mutex> lk(rt->mu);
        rt->stop = true;
        if (result == CVY_OK && !rt->err.empty()) result = CVY_E_STATE;
    }
    rt->cv_work.notify_all();
    rt->cv_driver.notify_all();
    poller.join();
    for (auto& w : workers) w.join();
    std::lock_guard<std::mutex> lk(rt->mu);
    for (Req& r : rt->reqs)
        if (r.submitted && !r.released) {
            if (!r.done) cvy_cancel_request(rt->e, r.rid);
            if (cvy_release_request(rt->e, r.rid) == CVY_OK) r.released = true;
        }
    rt->st.wall_s = rt->now();
    rt->st.driver_cpu_s = thread_cpu_s() - c0;
    if (result != CVY_OK) return cvy_internal_fail(result, rt->err);
    return CVY_OK;
}

cvy_status cvy_runtime_request_log(cvy_runtime* rt, uint32_t request, cvy_rt_request_log* out) {
    if (!rt || !out || request >= rt->reqs.size()) return cvy_internal_fail(CVY_E_INVAL, "runtime: bad request index");
    std::lock_guard<std::mutex> lk(rt->mu);
    const Req& r = rt->reqs[request];
    out->req_id = r.rid;
    out->t_arrival = r.t_arrival;
    out->t_submit = r.t_submit;
    out->t_done = r.t_done;
    out->t_abort = r.t_abort;
    out->n_rounds_run = (uint32_t)r.rounds.size();
    out->aborted = r.t_abort >= 0 ? 1u : 0u;
    return CVY_OK;
}

cvy_status cvy_runtime_round_log(cvy_runtime* rt, uint32_t request, uint32_t round, cvy_rt_round_log* out) {
    if (!rt || !out || request >= rt->reqs.size()) return cvy_internal_fail(CVY_E_INVAL, "runtime: bad request index");
    std::lock_guard<std::mutex> lk(rt->mu);
    const Req& r = rt->reqs[request];
    if (round >= r.rounds.size()) return cvy_internal_fail(CVY_E_INVAL, "runtime: bad round");
    out->t_start = r.rounds[round].t_start;
    out->t_final = r.rounds[round].t_final;
    out->n_pieces = (uint32_t)r.rounds[round].pieces.size();
    return CVY_OK;
}

cvy_status cvy_runtime_piece_log(cvy_runtime* rt, uint32_t request, uint32_t round, uint32_t piece,
                                 cvy_rt_piece_log* out) {
    if (!rt || !out || request >= rt->reqs.size()) return cvy_internal_fail(CVY_E_INVAL, "runtime: bad request index");
    std::lock_guard<std::mutex> lk(rt->mu);
    const Req& r = rt->reqs[request];
    if (round >= r.rounds.size() || piece >= r.rounds[round].pieces.size())
        return cvy_internal_fail(CVY_E_INVAL, "runtime: bad round / piece");
    const Piece& p = r.rounds[round].pieces[piece];
    out->t_avail = p.t_avail;
    out->t_dispatch = p.t_disp;
    out->t_begin = p.t_begin;
    out->t_end = p.t_end;
    out->cost_ms = p.plan.cost_ms;
    out->instance = p.plan.instance;
    out->token_index = p.token;
    out->n_deps = p.plan.n_deps;
    for (int k = 0; k < 8; ++k) out->deps[k] = p.plan.deps[k];
    return CVY_OK;
}

cvy_status cvy_runtime_stats(cvy_runtime* rt, cvy_rt_stats* out) {
    if (!rt || !out) return cvy_internal_fail(CVY_E_INVAL, "null argument");
    std::lock_guard<std::mutex> lk(rt->mu);
    *out = rt->st;
    return CVY_OK;
}

void cvy_runtime_destroy(cvy_runtime* rt) { delete rt; }
