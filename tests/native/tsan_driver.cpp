// Host-side race check of libconveyor's threading contract (include/conveyor.h): one thread
// steps the engine and releases finished requests, one consumer thread polls the segment
// ring (cvy_poll_segments: "exactly one consumer thread"), and a third thread submits and
// cancels requests concurrently (applied at the next step boundary).  Built with
// -fsanitize=thread together with a ThreadSanitizer build of libconveyor
// (scripts/tsan.sh); run on a B200.  A second phase runs the native runtime (cvy_runtime_*:
// driver, poller and executor threads) over 16 requests in both modes with aborts and refill.  Exit code 0 = contract exercised without errors;
// TSan reports go to stderr (halt_on_error=1 makes any race fatal).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "conveyor.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        cvy_status s_ = (x);                                                      \
        if (s_ != CVY_OK) {                                                       \
            std::fprintf(stderr, "%s -> %d: %s\n", #x, (int)s_, cvy_last_error()); \
            std::exit(2);                                                         \
        }                                                                         \
    } while (0)

int main() {
    cvy_model_config m{2, 128, 4, 2, 32, 384, 256, 1e-5f, 1e4, -1, CVY_DTYPE_BF16};  // the tiny parity config
    const uint32_t n_pages = 256;
    cvy_weight_sizes sz;
    CHECK(cvy_weight_sizes_for(&m, n_pages, &sz));
    size_t* szs = &sz.embed;
    void* bufs[10];
    for (int i = 0; i < 10; ++i) {
        if (cudaMalloc(&bufs[i], szs[i] ? szs[i] : 16) != cudaSuccess) return 3;
        cudaMemset(bufs[i], 0, szs[i] ? szs[i] : 16);
    }
    cvy_weights w{bufs[0], bufs[1], (const float*)bufs[2], (const float*)bufs[3], (const float*)bufs[4],
                  bufs[5], bufs[6], bufs[7], bufs[8], bufs[9]};
    CHECK(cvy_init_synthetic_weights(&m, &w, 1000, 0));
    cvy_engine_config ec{8, n_pages, 16, 1024, 4096, 512, 512, 512, 0, 0};
    std::vector<uint8_t> vb(256 * 16, 0), vl(256, 1);
    for (int i = 0; i < 256; ++i) vb[i * 16] = (uint8_t)i;
    cvy_engine* e = nullptr;
    CHECK(cvy_engine_create(&m, &ec, &w, vb.data(), vl.data(), &e));
    const uint8_t nl = '\n';
    const uint8_t* dl[1] = {&nl};
    const uint32_t dlen[1] = {1};
    cvy_tool_desc td{"python", CVY_PARSER_LITERAL, 1, dl, dlen, 0};
    int32_t tool = -1;
    CHECK(cvy_register_tool(e, &td, &tool));

    std::mutex mu;                    // guards live / finished (the driver's own state)
    std::vector<uint64_t> live;
    std::deque<uint64_t> finished;
    std::atomic<bool> stop{false};
    std::atomic<uint64_t> n_records{0}, n_final{0}, n_submitted{0}, n_cancel{0};
    const char* line = "x = 1\nprint(x)\n";
    std::vector<int32_t> forced;
    for (int r = 0; r < 4; ++r)
        for (const char* c = line; *c; ++c) forced.push_back((uint8_t)*c);

    auto submit = [&](uint64_t seed) {
        int32_t prompt[3] = {'#', ' ', '\n'};
        cvy_request_desc rd{};
        rd.tool_id = tool;
        rd.mode = CVY_MODE_PARTIAL;
        rd.prompt = prompt;
        rd.prompt_len = 3;
        rd.synth_prefix_len = (uint32_t)(seed % 20);
        rd.synth_seed = seed;
        rd.max_new_tokens = (uint32_t)forced.size();
        rd.forced = forced.data();
        rd.forced_len = (uint32_t)forced.size();
        uint64_t id = 0;
        cvy_status st = cvy_submit_request(e, &rd, &id);
        if (st == CVY_OK) {
            std::lock_guard<std::mutex> g(mu);
            live.push_back(id);
            n_submitted++;
        } else if (st != CVY_E_FULL) {
            std::fprintf(stderr, "submit: %d %s\n", (int)st, cvy_last_error());
            std::exit(4);
        }
    };

    // consumer: the single poller thread
    std::thread poller([&] {
        std::vector<cvy_segment> recs(256);
        std::vector<uint8_t> bytes(1 << 16);
        while (!stop.load()) {
            uint32_t n = 0;
            size_t used = 0;
            cvy_status st = cvy_poll_segments(e, recs.data(), (uint32_t)recs.size(), &n, bytes.data(), bytes.size(), &used);
            if (st == CVY_E_AGAIN) {
                std::this_thread::sleep_for(std::chrono::microseconds(50));
                continue;
            }
            if (st != CVY_OK) {
                std::fprintf(stderr, "poll: %d %s\n", (int)st, cvy_last_error());
                std::exit(5);
            }
            n_records += n;
            for (uint32_t i = 0; i < n; ++i)
                if (recs[i].flags & CVY_SEG_FINAL) {
                    n_final++;
                    std::lock_guard<std::mutex> g(mu);
                    finished.push_back(recs[i].req_id);
                }
        }
    });
    // submitter / canceller thread
    std::thread client([&] {
        std::mt19937_64 rng(7);
        uint64_t seed = 1;
        while (!stop.load()) {
            submit(seed++);
            uint64_t victim = 0;
            {
                std::lock_guard<std::mutex> g(mu);
                if (!live.empty() && rng() % 3 == 0) victim = live[rng() % live.size()];
            }
            if (victim) {
                cvy_status st = cvy_cancel_request(e, victim);
                if (st == CVY_OK) n_cancel++;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(300));
        }
    });
    // stepper: steps and releases finished requests
    for (int s = 0; s < 400; ++s) {
        cvy_step_info info{};
        CHECK(cvy_step(e, &info));
        std::deque<uint64_t> done;
        {
            std::lock_guard<std::mutex> g(mu);
            done.swap(finished);
        }
        for (uint64_t id : done) {
            if (cvy_request_state(e, id) == 0) {  // FINAL polled before the host saw the round end
                std::lock_guard<std::mutex> g(mu);
                finished.push_back(id);
                continue;
            }
            cvy_status st = cvy_release_request(e, id);
            if (st != CVY_OK && st != CVY_E_STATE) {
                std::fprintf(stderr, "release: %d %s\n", (int)st, cvy_last_error());
                return 6;
            }
            if (st == CVY_OK) {
                std::lock_guard<std::mutex> g(mu);
                for (size_t i = 0; i < live.size(); ++i)
                    if (live[i] == id) {
                        live.erase(live.begin() + (long)i);
                        break;
                    }
            }
        }
    }
    CHECK(cvy_sync(e));
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
    stop.store(true);
    client.join();
    poller.join();
    {
        // drain, then release everything still held so the native runtime below starts clean
        std::vector<cvy_segment> recs(256);
        uint32_t n = 0;
        size_t used = 0;
        while (cvy_poll_segments(e, recs.data(), (uint32_t)recs.size(), &n, nullptr, 0, &used) == CVY_OK) {
        }
        std::lock_guard<std::mutex> g(mu);
        for (uint64_t id : live) {
            cvy_cancel_request(e, id);
        }
        for (int s = 0; s < 4; ++s) CHECK(cvy_step(e, nullptr));
        CHECK(cvy_sync(e));
        while (cvy_poll_segments(e, recs.data(), (uint32_t)recs.size(), &n, nullptr, 0, &used) == CVY_OK) {
        }
        for (uint64_t id : live) cvy_release_request(e, id);
    }
    // the native runtime (cvy_runtime_*): its driver / poller / worker threads under TSan,
    // with a plan callback that aborts some requests and spreads pieces over 2 instances
    uint64_t rt_pieces = 0;
    for (int mode = 0; mode < 2; ++mode) {
        cvy_runtime_config rc{};
        rc.mode = mode == 0 ? CVY_MODE_PARTIAL : CVY_MODE_SEQUENTIAL;
        rc.n_workers = 4;
        rc.max_inflight = 4;
        rc.plan = [](void*, uint32_t request, uint32_t, uint32_t piece, const uint8_t*, uint32_t, uint16_t,
                     cvy_piece_plan* out) {
            out->cost_ms = 0.2;
            out->instance = (int32_t)(piece % 2);
            if (piece >= 2) {
                out->n_deps = 1;
                out->deps[0] = (int32_t)piece - 2;
            }
            out->abort = (request % 3 == 1 && piece == 3) ? 1 : 0;
        };
        cvy_runtime* rt = nullptr;
        CHECK(cvy_runtime_create(e, &rc, &rt));
        std::vector<cvy_round_desc> rounds(16);
        std::vector<cvy_rt_request> reqs(16);
        int32_t prompt[2] = {'#', '\n'};
        const int32_t obs[3] = {'o', 'k', '\n'};
        for (int i = 0; i < 16; ++i) {
            rounds[i] = cvy_round_desc{forced.data(), (uint32_t)forced.size(), tool, obs, 3};
            reqs[i] = cvy_rt_request{prompt, 2, (uint32_t)(i % 7), (uint64_t)i, &rounds[i], 1};
        }
        CHECK(cvy_runtime_run(rt, reqs.data(), 16, 120.0));
        cvy_rt_stats st{};
        CHECK(cvy_runtime_stats(rt, &st));
        rt_pieces += st.pieces;
        for (uint32_t i = 0; i < 16; ++i) {
            cvy_rt_request_log lg{};
            CHECK(cvy_runtime_request_log(rt, i, &lg));
            if (lg.t_done < lg.t_submit) return 8;
        }
        cvy_runtime_destroy(rt);
    }
    cvy_engine_destroy(e);
    for (void* b : bufs) cudaFree(b);
    std::printf("tsan driver ok: %llu submitted, %llu cancel calls, %llu records, %llu FINAL; native runtime: "
                "%llu pieces executed over 2 x 16 requests\n",
                (unsigned long long)n_submitted.load(), (unsigned long long)n_cancel.load(),
                (unsigned long long)n_records.load(), (unsigned long long)n_final.load(),
                (unsigned long long)rt_pieces);
    return n_final.load() > 0 ? 0 : 7;
}
