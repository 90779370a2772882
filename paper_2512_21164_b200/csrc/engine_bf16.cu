// Engine instantiation for u_s = bf16 (see engine.cuh).
#include "engine.cuh"
namespace gadi {
EngineVT engine_bf16 = Engine<bf16>::vt();
}  // namespace gadi
