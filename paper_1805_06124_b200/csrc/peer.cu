// peer.cu -- the PEER exchange wait (a4) of the column-sharded greedy.
//
// the parallel code exchanges the pivot information (MPI_Allreduce), sends
// the pivot column to the orthogonalising core (MPI_Send) and broadcasts the new basis vector
// (MPI_Bcast).  In the PEER mode every rank's sweep writes its 16-byte maxloc record straight
// into every rank's memory over NVLink (P2P stores, release-tagged) next to its candidate
// column in its own send slot; the replicated IMGS then reads the winner's column from the
// owner's slot over NVLink.  The only thing left between the two kernels is this wait for
// the world tags of the iteration -- no collective library call, no host round trip, CUDA-graph
// capturable.
#include "kernels.h"

namespace rbg {

__global__ void k_peer_wait(const PeerRec *mine, int world, DevState *st, unsigned long long epoch,
                            long long timeout_ns, cudaGraphConditionalHandle cond, int use_cond) {
    if (st->stop) {
        if (threadIdx.x == 0) loop_exit(cond, use_cond);
        return;
    }
    const unsigned long long tag = peer_tag(epoch, st->k);
    const int p = threadIdx.x;
    bool late = false;
    if (p < world) {
        const PeerRec *r = mine + ((st->k + 1) & 1) * world + p;
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(&r->tag) != tag) {
            if ((long long)(globaltimer_ns() - t0) > timeout_ns) {
                late = true;
                break;
            }
            __nanosleep(100);
        }
    }
    if (__any_sync(0xffffffffu, late) && p == 0) {
        st->stop = kStopPeer;
        loop_exit(cond, use_cond);
    }
}

cudaError_t launch_peer_wait(const PeerRec *mine, int world, DevState *st, unsigned long long epoch, long long timeout_ns,
                             cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s) {
    k_peer_wait<<<1, 32, 0, s>>>(mine, world, st, epoch, timeout_ns, cond, use_cond);
    return cudaGetLastError();
}

}  // namespace rbg
