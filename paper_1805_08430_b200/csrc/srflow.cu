// srflow.cu - libsrflow.so: the B200-native (sm_100a) transfer hot path.
//
// Host half: per-server HBM pools with the reference's region table, token
// and bounds gates (memspace.py:89-236), streams/events standing in for queue
// pairs and completion queues (fabric.py:113-143, :423-428), and the verb
// entry points (fabric.py:349-389).  Device half: the kernels K1..K6 of
// SURVEY.md section 2.2.  The reference moves bytes with a Python loop of
// 1-4096 B ascending chunks (fabric.py:391-421); here every byte moves through
// 16-byte vector loads/stores issued by all SMs, and the "final byte lands
// last" guarantee is rebuilt from a system-scope fence, a grid arrival count
// and one st.release.sys of the tail byte.
//
// Declarations and reference citations: include/srflow.h.

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/srflow.h"

namespace cg = cooperative_groups;

#include "host_objects.cuh"
#include "device_copy.cuh"
#include "device_pcg.cuh"
#include "device_ps.cuh"
#include "device_stream.cuh"
#include "device_rpc.cuh"
#include "host_record.cuh"
#include "host_launch.cuh"
#include "host_preload.cuh"
#include "abi_core.cuh"
#include "abi_ps.cuh"
#include "abi_stream.cuh"
#include "abi_doorbell.cuh"
