"""Exception classes of the transfer path.

Same names and the same inheritance as the reference hierarchy
(``errors.py:1-147`` of rdmaflow) so callers catching a reference class keep
working; the C ABI's status codes map onto these one to one
(``include/srflow.h``, ``_lib._STATUS``).  ``DeviceError`` is new: a CUDA
failure underneath a verb.
"""


class RdmaFlowError(Exception):
    """Root of every error raised by this package."""


def _family(name, base, doc):
    return type(name, (base,), {"__doc__": doc, "__module__": __name__})


# memory (reference errors.py:9-22)
ZeroLength = _family("ZeroLength", RdmaFlowError, "A zero-byte allocation or transfer.")
OutOfMemory = _family("OutOfMemory", RdmaFlowError, "Space capacity or region table exhausted.")
ArenaExhausted = _family("ArenaExhausted", RdmaFlowError, "No free arena block is large enough.")
OutOfBounds = _family("OutOfBounds", RdmaFlowError, "A byte range escapes its handle or space.")

# fabric (reference errors.py:27-64)
FabricError = _family("FabricError", RdmaFlowError, "Verb-level failure.")
PeerUnreachable = _family("PeerUnreachable", FabricError, "No listening peer / no NVLink path.")
NotRegistered = _family("NotRegistered", FabricError, "Local verb buffer is not registered.")
BadToken = _family("BadToken", FabricError, "Remote access token does not match.")
RemoteOutOfBounds = _family("RemoteOutOfBounds", FabricError,
                            "Remote range is not inside one registered region.")
InvalidLength = _family("InvalidLength", FabricError, "Zero-length verb.")
RecvBufferTooSmall = _family("RecvBufferTooSmall", FabricError,
                             "Posted receive cannot hold the message.")
NoPostedReceive = _family("NoPostedReceive", FabricError, "Send found no posted receive.")
Timeout = _family("Timeout", FabricError, "A blocking operation missed its deadline.")
HandlerMissing = _family("HandlerMissing", FabricError, "RPC target has no handler.")

# wire (reference errors.py:69-86)
WireError = _family("WireError", RdmaFlowError, "Encode/decode failure.")
RankZero = _family("RankZero", WireError, "Metadata needs rank >= 1.")
RankMismatch = _family("RankMismatch", WireError, "Decoded rank differs from the edge's rank.")
BadElemType = _family("BadElemType", WireError, "Unknown element-type code.")
LengthMismatch = _family("LengthMismatch", WireError, "Inconsistent encoded lengths.")

# graph (reference errors.py:91-104)
GraphError = _family("GraphError", RdmaFlowError, "Graph construction/analysis failure.")
ShapeMismatch = _family("ShapeMismatch", GraphError, "Conflicting dimensions.")
MissingAnnotation = _family("MissingAnnotation", GraphError, "Input node without a shape.")
InvalidConfig = _family("InvalidConfig", GraphError, "Unusable workload/session parameters.")

# tracing (reference errors.py:109-110)
UnknownAddress = _family("UnknownAddress", RdmaFlowError,
                         "A transferred address was never traced.")

# protocols (reference errors.py:115-132)
ProtocolError = _family("ProtocolError", RdmaFlowError, "Transfer-protocol violation.")
Deadlock = _family("Deadlock", ProtocolError, "Scheduler watchdog saw no progress.")
SizeMismatch = _family("SizeMismatch", ProtocolError, "Tensor size differs from the plan.")
RankChanged = _family("RankChanged", ProtocolError, "Rank changed on a fixed-rank edge.")
ReassemblyGap = _family("ReassemblyGap", ProtocolError, "A fragment went missing.")

# bench configuration (reference errors.py:137-147)
ConfigError = _family("ConfigError", RdmaFlowError, "Scenario-config failure (exit code 2).")
UnknownKey = _family("UnknownKey", ConfigError, "Unknown config key.")
BadValue = _family("BadValue", ConfigError, "Config value failed validation.")

# new: the device underneath a verb failed
DeviceError = _family("DeviceError", RdmaFlowError, "CUDA failure underneath a verb.")
