// Engine instantiation for u_s = fp16 (see engine.cuh).
#include "engine.cuh"
namespace gadi {
EngineVT engine_fp16 = Engine<fp16>::vt();
}  // namespace gadi
