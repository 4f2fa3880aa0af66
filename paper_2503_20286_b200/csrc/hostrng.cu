// Host-side replica of NumPy's Generator.permutation on the Philox bit generator
// (the per-generation shuffles of variation.py:52 and nsga3.py:204).
//
// The reference draws these permutations on the host, sequentially; at pop 200k
// NumPy spends ~13 ms per generation in them -- longer than the whole GPU
// generation -- so the generation loop would be host-bound.  This is the same
// algorithm, bit for bit, in native code:
//   permutation(n) = arange(n) shuffled by Fisher-Yates, i = n-1 .. 1:
//       j = random_interval(i): mask = smallest 2^k - 1 >= i; draw
//           next_uint32 (i <= 0xFFFFFFFF) until (draw & mask) <= i
//       swap(a[i], a[j])
//   next_uint32 (philox_next32): the high half of the previous 64-bit output
//       if one is pending (has_uint32), else a fresh output's low half (the high
//       half is kept pending);
//   next_uint64 (philox_next): buffered outputs of Philox4x64-10, counter
//       incremented with carry before each block.
// The state struct carries every field of NumPy's Philox state, so the host
// Generator is set to exactly the state NumPy would have after the call.
#include <stdint.h>
#include <string.h>

#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/temo_b200.h"

namespace {

struct HostPhilox {
    uint64_t ctr[4], key[2], buf[4];
    int pos;
    int has32;
    uint32_t u32;

    static inline void mulhilo(uint64_t a, uint64_t b, uint64_t &hi, uint64_t &lo) {
        const __uint128_t p = (__uint128_t)a * b;
        hi = (uint64_t)(p >> 64);
        lo = (uint64_t)p;
    }

    inline void block() {
        // counter += 1 with carry (philox_next)
        if (++ctr[0] == 0 && ++ctr[1] == 0 && ++ctr[2] == 0) ++ctr[3];
        uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
        uint64_t k0 = key[0], k1 = key[1];
        for (int r = 0; r < 10; ++r) {
            if (r) {
                k0 += 0x9E3779B97F4A7C15ull;
                k1 += 0xBB67AE8584CAA73Bull;
            }
            uint64_t h0, l0, h1, l1;
            mulhilo(0xD2E7470EE14C6C93ull, c0, h0, l0);
            mulhilo(0xCA5A826395121157ull, c2, h1, l1);
            c0 = h1 ^ c1 ^ k0;
            c1 = l1;
            c2 = h0 ^ c3 ^ k1;
            c3 = l0;
        }
        buf[0] = c0;
        buf[1] = c1;
        buf[2] = c2;
        buf[3] = c3;
        pos = 0;
    }

    inline uint64_t next64() {
        if (pos >= 4) block();
        return buf[pos++];
    }

    inline uint32_t next32() {
        if (has32) {
            has32 = 0;
            return u32;
        }
        const uint64_t v = next64();
        has32 = 1;
        u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
};

inline uint64_t interval(HostPhilox &g, uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xFFFFFFFFull) {
        while ((v = (g.next32() & mask)) > max) {
        }
    } else {
        while ((v = (g.next64() & mask)) > max) {
        }
    }
    return v;
}

void load(HostPhilox &g, const temo_philox_host *s) {
    memcpy(g.ctr, s->counter, sizeof g.ctr);
    memcpy(g.key, s->key, sizeof g.key);
    memcpy(g.buf, s->buffer, sizeof g.buf);
    g.pos = s->buffer_pos;
    g.has32 = s->has_uint32;
    g.u32 = s->uinteger;
}

void store(const HostPhilox &g, temo_philox_host *s) {
    memcpy(s->counter, g.ctr, sizeof g.ctr);
    memcpy(s->buffer, g.buf, sizeof g.buf);
    s->buffer_pos = g.pos;
    s->has_uint32 = g.has32;
    s->uinteger = g.u32;
}

// Bulk form of the same stream, 4 Philox blocks at a time (independent 128-bit multiply chains).

inline void philox4_blocks(const uint64_t ctr0[4], const uint64_t key[2], uint64_t out[4][4]) {
    uint64_t c[4][4];
    for (int b = 0; b < 4; ++b) {
        uint64_t x0 = ctr0[0] + (uint64_t)b, x1 = ctr0[1], x2 = ctr0[2], x3 = ctr0[3];
        if (x0 < ctr0[0] && ++x1 == 0 && ++x2 == 0) ++x3;  // carry of the + b
        c[b][0] = x0; c[b][1] = x1; c[b][2] = x2; c[b][3] = x3;
    }
    // two blocks at a time: 4 in flight need 16 state words + temporaries > x86-64's 16 GPRs
    // (spills; measured 40 vs 23 ns per block)
    for (int b0 = 0; b0 < 4; b0 += 2) {
    uint64_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        for (int b = b0; b < b0 + 2; ++b) {
            uint64_t h0, l0, h1, l1;
            HostPhilox::mulhilo(0xD2E7470EE14C6C93ull, c[b][0], h0, l0);
            HostPhilox::mulhilo(0xCA5A826395121157ull, c[b][2], h1, l1);
            const uint64_t n0 = h1 ^ c[b][1] ^ k0, n2 = h0 ^ c[b][3] ^ k1;
            c[b][0] = n0;
            c[b][1] = l1;
            c[b][2] = n2;
            c[b][3] = l0;
        }
    }
    }
    for (int b = 0; b < 4; ++b)
        for (int q = 0; q < 4; ++q) out[b][q] = c[b][q];
}

// The raw outputs of blocks [b0, b0 + nb) after counter `ctr` (block b has counter ctr + 1 + b),
// written as u32 pairs (low, high) -- the order next_uint32 consumes them.
void gen_blocks(const uint64_t ctr[4], const uint64_t key[2], int64_t b0, int64_t nb, uint32_t *w) {
    int64_t b = 0;
    for (; b + 4 <= nb; b += 4) {
        uint64_t base[4] = {ctr[0] + 1 + (uint64_t)(b0 + b), ctr[1], ctr[2], ctr[3]};
        if (base[0] < ctr[0] && ++base[1] == 0 && ++base[2] == 0) ++base[3];  // carry
        uint64_t out[4][4];
        philox4_blocks(base, key, out);
        for (int q = 0; q < 4; ++q)
            for (int t = 0; t < 4; ++t) {
                w[8 * (b + q) + 2 * t] = (uint32_t)out[q][t];
                w[8 * (b + q) + 2 * t + 1] = (uint32_t)(out[q][t] >> 32);
            }
    }
    for (; b < nb; ++b) {
        HostPhilox h;
        for (int t = 0; t < 4; ++t) h.ctr[t] = ctr[t];
        h.key[0] = key[0];
        h.key[1] = key[1];
        uint64_t add = (uint64_t)(b0 + b);
        // counter + (b0 + b) with carry, then block() adds the final + 1
        const uint64_t c0 = h.ctr[0];
        h.ctr[0] += add;
        if (h.ctr[0] < c0 && ++h.ctr[1] == 0 && ++h.ctr[2] == 0) ++h.ctr[3];
        h.block();
        for (int t = 0; t < 4; ++t) {
            w[8 * b + 2 * t] = (uint32_t)h.buf[t];
            w[8 * b + 2 * t + 1] = (uint32_t)(h.buf[t] >> 32);
        }
    }
}

// Persistent worker threads for the block generation (spawning threads per call cost ~1 ms of
// the ~3 ms permutation at n = 400k).  Re-created after fork (pid check).
struct Pool {
    std::mutex call;  // one run at a time (the host pipeline thread and the caller may both draw)
    std::mutex mu;
    std::condition_variable cv, done;
    const uint64_t *ctr = nullptr, *key = nullptr;
    int64_t base = 0, per = 0, end = 0;
    uint32_t *w = nullptr;
    uint64_t round = 0;
    int T = 0, pending = 0;
    pid_t pid = 0;

    void start(int nt) {
        T = nt;
        pid = getpid();
        for (int t = 0; t < T; ++t) std::thread([this, t] { loop(t); }).detach();
    }
    void loop(int t) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return round != seen; });
            seen = round;
            const int64_t s0 = base + t * per;
            const int64_t cnt = s0 + per <= end ? per : end - s0;
            const uint64_t *c = ctr, *k = key;
            uint32_t *out = w;
            lk.unlock();
            if (cnt > 0) gen_blocks(c, k, s0, cnt, out + 8 * s0);
            lk.lock();
            if (--pending == 0) done.notify_one();
        }
    }
    // blocks [b0, b1) of the stream into w (the calling thread waits)
    void run(const uint64_t *c, const uint64_t *k, int64_t b0, int64_t b1, uint32_t *out) {
        std::lock_guard<std::mutex> one(call);
        std::unique_lock<std::mutex> lk(mu);
        ctr = c;
        key = k;
        base = b0;
        end = b1;
        per = ((b1 - b0 + T - 1) / T + 3) / 4 * 4;
        w = out;
        pending = T;
        ++round;
        cv.notify_all();
        done.wait(lk, [&] { return pending == 0; });
    }
};

static Pool *pool() {
    static Pool *p = nullptr;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    if (!p || p->pid != getpid()) {  // first use, or a forked child (the threads are gone)
        int T = (int)std::thread::hardware_concurrency();
        if (T > 8) T = 8;
        if (T < 2) return nullptr;
        p = new Pool();  // leaked on purpose: detached workers may outlive static destruction
        p->start(T);
    }
    return p;
}

// grow-only u32 buffer, reused across calls by the calling thread (no zero-fill, no page faults)
struct Words {
    std::unique_ptr<uint32_t[]> p;
    size_t cap = 0;
    uint32_t *grow(size_t n, size_t keep) {
        if (n > cap) {
            std::unique_ptr<uint32_t[]> q(new uint32_t[n + n / 4]);
            if (keep) memcpy(q.get(), p.get(), keep * sizeof(uint32_t));
            p.swap(q);
            cap = n + n / 4;
        }
        return p.get();
    }
};

// A window of the u32 stream of g, generated ahead in parallel (counter-based, so any
// block is independent); `take` hands out values in order and `commit` leaves g exactly
// where NumPy's Generator would be after the consumed values.
struct Stream32 {
    HostPhilox &g;
    std::vector<uint32_t> head;  // pending high half + rest of the current buffer
    uint32_t *w = nullptr;       // whole blocks after the buffer (thread-local reused storage)
    int64_t nb = 0, pos = 0;     // blocks generated, u32 consumed (head first)
    static Words &store() {
        thread_local Words ws;
        return ws;
    }

    explicit Stream32(HostPhilox &gg) : g(gg) {
        if (g.has32) head.push_back(g.u32);
        for (int q = g.pos; q < 4; ++q) {
            head.push_back((uint32_t)g.buf[q]);
            head.push_back((uint32_t)(g.buf[q] >> 32));
        }
    }

    void ensure(int64_t total) {  // at least `total` u32 available
        const int64_t need_blocks = (total - (int64_t)head.size() + 7) / 8;
        if (need_blocks <= nb) return;
        const int64_t nb2 = need_blocks > nb + nb / 2 ? need_blocks : nb + nb / 2 + 1024;
        w = store().grow((size_t)nb2 * 8, (size_t)nb * 8);
        const int64_t add = nb2 - nb;
        Pool *P = add < 4096 ? nullptr : pool();
        if (!P) gen_blocks(g.ctr, g.key, nb, add, w + 8 * nb);
        else P->run(g.ctr, g.key, nb, nb2, w);
        nb = nb2;
    }

    inline uint32_t at(int64_t k) const {
        return k < (int64_t)head.size() ? head[(size_t)k] : w[(size_t)(k - (int64_t)head.size())];
    }

    void commit(int64_t used) {  // the Generator state after `used` next_uint32 calls
        int64_t k = used;
        const int64_t h0 = g.has32 ? 1 : 0;
        if (k <= h0) {
            if (k == 1) g.has32 = 0;
            return;
        }
        k -= h0;  // u32 drawn from 64-bit outputs
        const int64_t words = (k + 1) / 2;
        const bool odd = k & 1;
        const int64_t inbuf = 4 - g.pos;
        uint32_t hi = 0;
        if (words <= inbuf) {
            hi = (uint32_t)(g.buf[g.pos + words - 1] >> 32);
            g.pos += (int)words;
        } else {
            const int64_t rest = words - inbuf;           // words from new blocks
            const int64_t blocks = (rest + 3) / 4;
            const int64_t last = blocks - 1;              // last block touched
            for (int q = 0; q < 4; ++q)
                g.buf[q] = (uint64_t)w[(size_t)(8 * last + 2 * q)] | ((uint64_t)w[(size_t)(8 * last + 2 * q + 1)] << 32);
            const uint64_t c0 = g.ctr[0];
            g.ctr[0] += (uint64_t)blocks;
            if (g.ctr[0] < c0 && ++g.ctr[1] == 0 && ++g.ctr[2] == 0) ++g.ctr[3];
            g.pos = (int)(rest - 4 * last);
            hi = (uint32_t)(g.buf[g.pos - 1] >> 32);
        }
        g.has32 = odd ? 1 : 0;
        g.u32 = hi;  // NumPy keeps the last high half in uinteger even once it is consumed
    }
};

}  // namespace

extern "C" int temo_host_permutation(temo_philox_host *st, int64_t n, int64_t *out) {
    if (!st || n < 0 || (n > 0 && !out) || st->buffer_pos < 0 || st->buffer_pos > 4) return TEMO_EINVAL;
    HostPhilox g;
    load(g, st);
    if (n > 1 && n <= INT32_MAX) {
        // 1) draws: the u32 stream generated ahead in parallel, consumed by the rejection
        //    automaton one mask class at a time (branch-free: j_i is rewritten until accepted);
        // 2) swaps: random accesses on an int32 work array, j prefetched ahead.
        int32_t *a = reinterpret_cast<int32_t *>(out);             // out[0 .. n/2): work array
        int32_t *js = a + n;                                       // out[n/2 .. n): j_i (i >= 1)
        Stream32 S(g);
        int64_t p = 0;
        int64_t i = n - 1;
        S.ensure(n + n / 2 + 64);
        // 3) the swaps run on a second thread behind the automaton: js[k] is final once the
        //    automaton's i has moved below k (published as `frontier`, release/acquire)
        std::atomic<int64_t> frontier(n - 1);
        auto swaps = [&] {
            for (int64_t k = 0; k < n; ++k) a[k] = (int32_t)k;
            constexpr int64_t PF = 32;
            int64_t k = n - 1;
            while (k >= 1) {
                int64_t f;
                while ((f = frontier.load(std::memory_order_acquire)) >= k) std::this_thread::yield();
                for (; k > f && k >= 1; --k) {
                    if (k - PF > f) __builtin_prefetch(a + js[k - PF], 1, 3);
                    const int64_t j = js[k];
                    const int32_t t = a[j];
                    a[j] = a[k];
                    a[k] = t;
                }
            }
            for (int64_t q = n - 1; q >= 0; --q) out[q] = (int64_t)a[q];  // widen (back to front)
        };
        const bool two = n >= (1 << 16) && std::thread::hardware_concurrency() >= 2;
        std::thread sw;
        if (two) sw = std::thread(swaps);
        while (i >= 1) {
            const int lz = __builtin_clzll((uint64_t)i);
            const uint32_t mask = (uint32_t)(~0ull >> lz);
            const int64_t lo = (int64_t)(mask >> 1);                 // the class ends when i == lo
            while (i > lo) {
                S.ensure(p + 2 * (i - lo) + 64);
                const int64_t pend = p + (i - lo);                   // draws surely consumed
                const int64_t cap = (int64_t)S.head.size() + 8 * S.nb;
                const int64_t stop = pend < cap ? pend : cap;
                while (p < stop) {  // at least `stop - p` more acceptances are needed: no overrun
                    const int64_t lim = stop - p > 8192 ? p + 8192 : stop;
                    while (p < lim) {
                        const uint32_t v = S.at(p++) & mask;
                        js[i] = (int32_t)v;
                        i -= (int64_t)(v <= (uint32_t)i);
                    }
                    frontier.store(i, std::memory_order_release);
                }
            }
        }
        frontier.store(0, std::memory_order_release);
        S.commit(p);
        if (two) sw.join();
        else swaps();
    } else {
        for (int64_t k = 0; k < n; ++k) out[k] = k;
        for (int64_t k = n - 1; k >= 1; --k) {
            const int64_t j = (int64_t)interval(g, (uint64_t)k);
            const int64_t t = out[j];
            out[j] = out[k];
            out[k] = t;
        }
    }
    store(g, st);
    return TEMO_OK;
}
