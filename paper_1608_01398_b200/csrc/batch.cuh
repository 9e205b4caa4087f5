// Internal: lock-step batching of concurrent fits' X^T r sweeps (batch.cu).
#pragma once

#include "handle.cuh"

struct gi_batch;
// the calling fit is live in the group from join to leave
int gi_batch_join(gi_batch* b);
int gi_batch_leave(gi_batch* b);
// hand this fit's right-hand side to the group (ready once `s` reaches this
// point) and block until the sweep that serves it has been launched; `s`
// then waits on that sweep (through the fit's own `done` event)
int gi_batch_submit(gi_batch* b, const gi::XtrRhs& rhs, cudaStream_t s, cudaEvent_t ready,
                    cudaEvent_t done);
bool gi_batch_matches(const gi_batch* b, const gi_matrix* h);
