// Engine instantiation for u_s = fp32 (see engine.cuh).
#include "engine.cuh"
namespace gadi {
EngineVT engine_fp32 = Engine<float>::vt();
}  // namespace gadi
