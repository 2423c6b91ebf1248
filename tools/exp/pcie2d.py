import torch, time, ctypes, glob, os
import nvidia.cuda_runtime as cr
lib = glob.glob(os.path.join(os.path.dirname(cr.__file__ if cr.__file__ else list(cr.__path__)[0]), "lib", "libcudart.so*"))
rt = ctypes.CDLL(lib[0])
n = 192 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
for width, pitch in ((256, 8192), (1024, 4096), (1024, 8192), (2048, 8192), (4096, 8192), (8192, 16384)):
    rows = n // pitch
    f = lambda: rt.cudaMemcpy2DAsync(ctypes.c_void_p(d.data_ptr()), ctypes.c_size_t(pitch), ctypes.c_void_p(h.data_ptr()), ctypes.c_size_t(pitch), ctypes.c_size_t(width), ctypes.c_size_t(rows), 1, ctypes.c_void_p(st))
    tt = t(f)
    print(f"cudaMemcpy2DAsync H2D width {width} B pitch {pitch}: {rows*width/tt/1e9:.1f} GB/s")
