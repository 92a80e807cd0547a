// Native request-storm driver for BASELINE config 4 (bench.py, tests): N
// client threads stand in for N cafx client actors and push requests into one
// compute actor through cafxg_actor_enqueue (the seam an adapter actor's
// `enqueue` forwards to, abstract_actor.hpp:36).
//
//  * open loop  (mode 0): every client sends all its requests back to back,
//    replies directed to the sender (async `send`, local_actor.cpp:325-327);
//  * closed loop (mode 1): one outstanding request per client, the
//    `sync_send(...).then(...)` discipline (local_actor.cpp:99-101), one OS
//    thread per client blocked on its reply;
//  * closed loop on a scheduler (mode 2): the same discipline with the
//    clients multiplexed over W worker threads the way cafx runs actors
//    (scheduler.hpp:24-45: CAFX_WORKERS, default hardware_concurrency). A reply
//    makes its client runnable on its worker (the mailbox enqueue that
//    schedules an actor); the worker runs the `.then` continuation, which
//    sends the client's next request.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/cafxg.h"

namespace {

struct Client {
  std::atomic<uint32_t> done{0};  // replies received (C++20 atomic wait)
  std::atomic<uint32_t>* errors;
};

// Runs on a libcafxg completion/callback thread: one atomic increment and a
// futex wake only when the client is actually waiting.
void on_done(void* user, int status) {
  auto* c = static_cast<Client*>(user);
  if (status != CAFXG_OK)
    c->errors->fetch_add(1);
  c->done.fetch_add(1, std::memory_order_release);
  c->done.notify_one();
}

void wait_for(Client& c, uint32_t n) {
  uint32_t v = c.done.load(std::memory_order_acquire);
  while (v < n) {
    c.done.wait(v, std::memory_order_acquire);
    v = c.done.load(std::memory_order_acquire);
  }
}

// Mode 2: a worker's run queue of clients whose reply arrived.
struct Worker {
  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint32_t> ready;
  bool sleeping = false;
};

struct SchedClient {
  Worker* w;
  uint32_t id;
  uint32_t sent = 0;
  std::atomic<uint32_t>* errors;
};

void on_done_sched(void* user, int status) {
  auto* c = static_cast<SchedClient*>(user);
  if (status != CAFXG_OK)
    c->errors->fetch_add(1);
  Worker* w = c->w;
  bool wake;
  {
    std::lock_guard<std::mutex> g(w->mu);
    w->ready.push_back(c->id);
    wake = w->sleeping;
  }
  if (wake)
    w->cv.notify_one();
}

int run_scheduled(cafxg_actor* actor, const cafxg_mandel_desc* descs, uint8_t* replies,
                  size_t reply_bytes, uint32_t clients, uint32_t per,
                  std::atomic<uint32_t>& errors) {
  const char* e = getenv("CAFX_WORKERS");
  uint32_t nw = e && atoi(e) > 0 ? (uint32_t)atoi(e) : std::thread::hardware_concurrency();
  nw = std::max<uint32_t>(1, std::min(nw, clients));
  std::vector<Worker> ws(nw);
  std::vector<SchedClient> cs(clients);
  for (uint32_t c = 0; c < clients; ++c) {
    cs[c].w = &ws[c % nw];
    cs[c].id = c;
    cs[c].errors = &errors;
    ws[c % nw].ready.push_back(c);  // every client starts runnable
  }
  std::atomic<int> status{CAFXG_OK};
  std::vector<std::thread> th;
  for (uint32_t wi = 0; wi < nw; ++wi) {
    th.emplace_back([&, wi] {
      Worker& w = ws[wi];
      uint32_t mine = 0;  // clients of this worker that sent everything
      const uint32_t owned = (clients - wi + nw - 1) / nw;
      std::vector<uint32_t> run;
      size_t sz = sizeof(cafxg_mandel_desc);
      while (mine < owned) {
        {
          std::unique_lock<std::mutex> lk(w.mu);
          while (w.ready.empty()) {
            w.sleeping = true;
            w.cv.wait(lk);
            w.sleeping = false;
          }
          run.swap(w.ready);
        }
        for (uint32_t c : run) {
          SchedClient& me = cs[c];
          if (me.sent == per) {  // last reply in
            ++mine;
            continue;
          }
          uint64_t k = (uint64_t)c * per + me.sent++;
          const void* in[1] = {&descs[k]};
          int s = cafxg_actor_enqueue(actor, in, &sz, 1, replies + k * reply_bytes,
                                      reply_bytes, on_done_sched, &me);
          if (s != CAFXG_OK) {
            status.store(s);
            me.sent = per;
            ++mine;
          }
        }
        run.clear();
      }
    });
  }
  for (auto& t : th)
    t.join();
  return status.load();
}

}  // namespace

extern "C" {

// descs: clients*per descriptors (request k = client k/per); replies: one
// reply buffer of `reply_bytes` per request, contiguous. Returns 0 and fills
// wall_ms / errors, or the first enqueue failure status.
int cafxg_storm_run(cafxg_actor* actor, const cafxg_mandel_desc* descs,
                    uint8_t* replies, size_t reply_bytes, uint32_t clients,
                    uint32_t per, int closed_loop, double* wall_ms,
                    uint32_t* errors_out) {
  std::atomic<uint32_t> errors{0};
  std::atomic<int> enqueue_status{CAFXG_OK};
  std::vector<Client> cs(clients);
  for (auto& c : cs)
    c.errors = &errors;
  const uint64_t total = (uint64_t)clients * per;
  auto t0 = std::chrono::steady_clock::now();
  if (closed_loop == 2) {
    int s = run_scheduled(actor, descs, replies, reply_bytes, clients, per, errors);
    auto t1 = std::chrono::steady_clock::now();
    if (wall_ms)
      *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (errors_out)
      *errors_out = errors.load();
    return s;
  }
  std::vector<std::thread> th;
  th.reserve(clients);
  for (uint32_t c = 0; c < clients; ++c) {
    th.emplace_back([&, c] {
      Client& me = cs[c];
      size_t sz = sizeof(cafxg_mandel_desc);
      for (uint32_t i = 0; i < per; ++i) {
        uint64_t k = (uint64_t)c * per + i;
        const void* in[1] = {&descs[k]};
        int s = cafxg_actor_enqueue(actor, in, &sz, 1, replies + k * reply_bytes,
                                    reply_bytes, on_done, &me);
        if (s != CAFXG_OK) {
          enqueue_status.store(s);
          return;
        }
        if (closed_loop)
          wait_for(me, i + 1);
      }
      wait_for(me, per);
    });
  }
  for (auto& t : th)
    t.join();
  auto t1 = std::chrono::steady_clock::now();
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  if (errors_out)
    *errors_out = errors.load();
  (void)total;
  return enqueue_status.load();
}

}  // extern "C"
