// Device side of the pipeline timeline: the "gap" kernel that stands in for
// a stage's receive of its cross-stage dependency (replica mode) and reports
// bubble boundaries to the host worker through a mapped event ring -- the
// role the paper's three DeepSpeed instrumentation points play
// (PAPER.md:643-647): BubbleStarted when the preceding op on the stage
// completes, BubbleEnded when the next op becomes ready.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace freeride::rt {

// One slot of the host-mapped event ring.  The device writes t/code then
// publishes `seq` (slot index + 1) after a system-scope fence.
struct alignas(16) RingSlot {
  std::uint64_t t_ns;  // %globaltimer
  std::uint32_t code;  // see ring_code()
  std::uint32_t seq;
};

enum : std::uint32_t { kEvBubbleStart = 1u, kEvBubbleEnd = 2u, kEvEpochBase = 3u };

inline std::uint32_t ring_code(std::uint32_t kind, std::uint32_t bubble) {
  return (kind << 28) | (bubble & 0x0FFFFFFFu);
}

struct TimelineCtl {
  std::uint64_t base_ns;   // start of the current epoch (device clock)
  std::uint64_t last_ns;
  std::uint32_t end_seq;   // token of the last bubble that ended (imperative preemption)
  std::uint32_t link_timeouts;  // linked waits that gave up (neighbour never signalled)
  std::uint64_t run0_ns;        // the run's first gap (device clock): origin of the run's records
};

struct GapArgs {
  TimelineCtl* ctl;
  RingSlot* ring;            // host-mapped
  std::uint32_t ring_mask;
  std::int64_t slot_start;   // -1: no event
  std::int64_t slot_end;     // -1: no event
  std::uint32_t code_start;
  std::uint32_t code_end;
  std::int64_t ready_ns;     // dependency ready, relative to the epoch base
  std::int64_t span_ns;      // epoch span (epoch-end gaps)
  std::int32_t mode;         // 0: before an op, 1: epoch end, 2: first epoch begin
  std::uint32_t end_token;   // > 0: raise ctl->end_seq to this at the bubble end
};

// Peer-linked pipeline (transport 1): the wait for a cross-stage dependency
// is a spin on this stage's own mailbox flag, which the neighbouring stage
// raises (over NVLink / peer memory) after its copy of the activation or
// gradient into this stage's mailbox slot has completed.
struct LinkWaitArgs {
  TimelineCtl* ctl;
  RingSlot* ring;
  std::uint32_t ring_mask;
  std::int64_t slot_start;     // -1: no event
  std::int64_t slot_end;
  std::uint32_t code_start;
  std::uint32_t code_end;
  const std::uint32_t* flag;   // null: nothing to wait for
  std::uint32_t seq;           // wait until *flag >= seq
  std::uint32_t end_token;
  std::int32_t mode;           // 2: first gap of the run (sets the epoch base)
  std::uint64_t timeout_ns;    // give up (and count it) after this long
};

void launch_link_wait(const LinkWaitArgs& a, cudaStream_t s);
// *flag = v (release, system scope) once the preceding stream work is done
void launch_link_signal(std::uint32_t* flag, std::uint32_t v, cudaStream_t s);

void configure_timeline_kernels();
// preferred L1/shared split (percent) of the gap / link / stamp kernels
void set_wait_kernel_carveout(int percent);
void launch_gap(const GapArgs& a, cudaStream_t s);
// Writes %globaltimer to *host_mapped and publishes it through *flag.
void launch_stamp(std::uint64_t* host_mapped, volatile std::uint32_t* flag, std::uint32_t val,
                  cudaStream_t s);

}  // namespace freeride::rt
