# libspl: B200 (sm_100a) sequence-parallel layer. `make -j` builds the shared library in-tree
# (it travels to the GPU box with the gpurun snapshot) plus the oracle checker.
NVCC ?= /usr/local/cuda/bin/nvcc
# NCCL: the torch-bundled 2.28 (same soname libnccl.so.2 as the system 2.27) so that libspl and
# torch share one NCCL in a process whichever loads first.
NCCL_HOME ?= $(shell python -c "import nvidia.nccl as n; print(list(n.__path__)[0])" 2>/dev/null)
ifeq ($(NCCL_HOME),)
NCCL_INC :=
NCCL_LINK := -lnccl
else
NCCL_INC := -I$(NCCL_HOME)/include
NCCL_LINK := -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_HOME)/lib
endif
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Iinclude $(NCCL_INC) -Xptxas -warn-spills
PKG := paper_2205_05198_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.hpp $(PKG)/csrc/*.cuh) include/spl.h

all: $(PKG)/libspl.so oracle build/test_facade build/test_window_facade

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libspl.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) $(NCCL_LINK)

build/test_facade: tests/cpp/test_facade.cpp include/spl_seqpar.hpp include/spl.h $(PKG)/libspl.so
	g++ -std=c++20 -O2 -Wall -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -lspl \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

build/test_window_facade: tests/cpp/test_window_facade.cpp include/spl_pipeline.hpp include/spl.h $(PKG)/libspl.so
	g++ -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(PKG) -lspl -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libspl.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
