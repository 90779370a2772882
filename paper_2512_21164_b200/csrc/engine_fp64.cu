// Engine instantiation for u_s = fp64 (see engine.cuh).
#include "engine.cuh"
namespace gadi {
EngineVT engine_fp64 = Engine<double>::vt();
}  // namespace gadi
