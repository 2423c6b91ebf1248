# Top-level build: the product library (sm_100a CUDA + C ABI + C++ adapter)
# and the oracle (test infrastructure).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2312_11918_b200
LIB := $(PKG)/libfmha_b200.so
SRCS := $(PKG)/csrc/fmha_api.cu $(PKG)/csrc/fmha_reference.cu $(PKG)/csrc/fmha_host.cpp $(PKG)/csrc/fmha_io.cpp
HDRS := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.hpp include/fmha/*.h include/fmha/*.hpp)

CLI := $(PKG)/fmha-b200

all: $(LIB) $(CLI) oracle

# the C++ CLI (reference fmha-sim counterpart), linked against the library
$(CLI): $(PKG)/csrc/fmha_cli.cpp $(LIB) include/fmha/fmha.h include/fmha/fmha.hpp
	$(NVCC) -std=c++20 -O2 -o $@ $(PKG)/csrc/fmha_cli.cpp -L$(PKG) -lfmha_b200 -Xlinker -rpath -Xlinker '$$ORIGIN'


$(PKG)/csrc/tmem_ops.cuh: tools/gen_tmem_ops.py
	python tools/gen_tmem_ops.py

$(LIB): $(SRCS) $(HDRS) $(PKG)/csrc/tmem_ops.cuh
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -lpthread 2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "registers|spill|smem" build/ptxas.log | sed 's/^/  /' || true

# timeline-instrumented build for tools/trace_timeline.py (FMHA_B200_LIB selects it)
trace: build/libfmha_b200_trace.so
build/libfmha_b200_trace.so: $(SRCS) $(HDRS) $(PKG)/csrc/tmem_ops.cuh | build
	$(NVCC) $(NVFLAGS) -DFMHA_TRACE_BUILD -shared -o $@ $(SRCS) -lpthread 2> build/ptxas_trace.log || (cat build/ptxas_trace.log; false)

# phase-profile build for tools/prof_phases.py (FMHA_B200_LIB selects it)
prof: build/libfmha_b200_prof.so
build/libfmha_b200_prof.so: $(SRCS) $(HDRS) $(PKG)/csrc/tmem_ops.cuh | build
	$(NVCC) $(NVFLAGS) -DFMHA_PROF_BUILD -shared -o $@ $(SRCS) -lpthread 2> build/ptxas_prof.log || (cat build/ptxas_prof.log; false)

# watchdog build (mbarrier waits trap after ~4 s): tests of risky kernel changes,
# tools/sanitize_smoke.py; FMHA_B200_LIB=build/libfmha_b200_watchdog.so selects it
watchdog: build/libfmha_b200_watchdog.so
build/libfmha_b200_watchdog.so: $(SRCS) $(HDRS) $(PKG)/csrc/tmem_ops.cuh | build
	$(NVCC) $(NVFLAGS) -DFMHA_WATCHDOG -shared -o $@ $(SRCS) -lpthread 2> build/ptxas_watchdog.log || (cat build/ptxas_watchdog.log; false)

oracle:
	$(MAKE) -s -C oracle all

build/ptxas.log: | build
build:
	mkdir -p build

$(LIB): | build

clean:
	rm -f $(LIB) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean trace watchdog prof
