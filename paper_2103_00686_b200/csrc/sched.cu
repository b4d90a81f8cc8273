// sched.cu — the hot/cold scheduler (§4.3,
// P:L538-572, Eq. 5).  Host-only: the interleaving of the cold
// and hot mini-batch queues of an epoch and the loss-feedback rate r(i).
// Readings R28-R31, restated in include/fae.h.
#include <cmath>

#include "fae_internal.cuh"

extern "C" {

fae_status fae_sched_init(fae_sched* s, int64_t n_cold, int64_t n_hot, double r_start, int32_t u) {
    if (!s || n_cold < 0 || n_hot < 0 || !(r_start >= 1.0 && r_start <= 100.0) || u < 1 || u > FAE_SCHED_MAX_U)
        return FAE_ERR_INVALID_ARG;
    *s = fae_sched{};
    s->n[FAE_SCHED_COLD] = n_cold;
    s->n[FAE_SCHED_HOT] = n_hot;
    s->r = r_start;
    s->u = u;
    s->next_kind = FAE_SCHED_COLD;   // P:L543 "always begins with training on cold inputs"
    s->last_kind = -1;
    return FAE_OK;
}

fae_status fae_sched_new_epoch(fae_sched* s) {
    if (!s) return FAE_ERR_INVALID_ARG;
    s->done[0] = s->done[1] = 0;
    s->next_kind = FAE_SCHED_COLD;
    s->last_kind = -1;
    return FAE_OK;
}

fae_status fae_sched_next(fae_sched* s, int32_t* kind, int64_t* first, int64_t* count, int32_t* swap_after) {
    if (!s || !kind || !first || !count || !swap_after) return FAE_ERR_INVALID_ARG;
    int k = s->next_kind, o = 1 - k;
    *count = 0;
    *first = 0;
    *swap_after = 0;
    *kind = k;
    if (s->done[k] >= s->n[k]) {
        k = o;
        o = 1 - k;
        if (s->done[k] >= s->n[k]) return FAE_OK;   // both drained
    }
    const int64_t left = s->n[k] - s->done[k];
    // R(r): ceil(r% of the kind's original count), at least one batch
    int64_t len = (int64_t)std::ceil(s->r / 100.0 * (double)s->n[k]);
    if (len < 1) len = 1;
    const int64_t cnt = s->done[o] >= s->n[o] ? left : (len < left ? len : left);
    *kind = k;
    *first = s->done[k];
    *count = cnt;
    s->done[k] += cnt;
    s->next_kind = o;
    s->last_kind = k;
    *swap_after = s->done[o] < s->n[o] ? 1 : 0;
    return FAE_OK;
}

fae_status fae_sched_record_swap(fae_sched* s, double test_loss, int64_t hot_bytes, int32_t n_devices) {
    if (!s || !std::isfinite(test_loss) || n_devices < 1 || hot_bytes < 0) return FAE_ERR_INVALID_ARG;
    s->swaps++;
    s->sync_events += n_devices;          // each change of kind syncs the hot rows
    s->sync_bytes += hot_bytes * n_devices;
    // keep the last u + 1 losses (oldest first)
    if (s->n_hist == s->u + 1) {
        for (int i = 1; i < s->n_hist; i++) s->hist[i - 1] = s->hist[i];
        s->n_hist--;
    }
    s->hist[s->n_hist++] = test_loss;
    const int h = s->n_hist;
    if (h < 2) return FAE_OK;                               // no predecessor: unchanged
    if (s->hist[h - 1] > s->hist[h - 2]) {                  // Eq. 5 case 1: halve, clamp at R(1)
        s->r = s->r / 2.0 < 1.0 ? 1.0 : s->r / 2.0;
        return FAE_OK;
    }
    if (h == s->u + 1) {                                    // case 2: u successive decreases
        bool dec = true;
        for (int i = 1; i < h; i++) dec = dec && s->hist[i] < s->hist[i - 1];
        if (dec) s->r = s->r * 2.0 > 100.0 ? 100.0 : s->r * 2.0;
    }
    return FAE_OK;                                          // case 3: unchanged
}

}  // extern "C"
