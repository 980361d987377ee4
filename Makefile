# Build the C-ABI library without Python (the same flags as __graft_entry__.build()).
#   make            -> paper_1902_05234_b200/libaes_b200.so, synth/libsynth.so, oracle/liboracle.so
#   make c-test     -> tests/c/test_abi (plain-C user of include/aes_b200.h); run with `gpu` on a B200
NVCC  ?= /usr/local/cuda/bin/nvcc
ARCH  := -gencode arch=compute_100a,code=sm_100a
FLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Iinclude
PKG   := paper_1902_05234_b200
SRC   := $(PKG)/csrc/aes_ecb.cu $(PKG)/csrc/aes_batch.cu $(PKG)/csrc/aes_runtime.cu \
         $(PKG)/csrc/aes_pipeline.cu $(PKG)/csrc/aes_keysched.cpp
HDR   := include/aes_b200.h $(PKG)/csrc/aes_tables.h $(PKG)/csrc/aes_device.cuh $(PKG)/csrc/aes_host.h
OBJ   := $(patsubst %,build/%.o,$(notdir $(SRC)))

all: $(PKG)/libaes_b200.so synth/libsynth.so oracle/liboracle.so

build/%.o: $(PKG)/csrc/% $(HDR)
	@mkdir -p build
	$(NVCC) $(FLAGS) -c -o $@ $<

$(PKG)/libaes_b200.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $^

synth/libsynth.so: synth/fill.cu
	$(NVCC) $(FLAGS) -shared -o $@ $<

oracle/liboracle.so: oracle/aes_oracle.c
	gcc -O2 -std=c11 -fPIC -fno-semantic-interposition -shared -pthread -o $@ $<

c-test: $(PKG)/libaes_b200.so tests/c/test_abi.c
	gcc -std=c11 -O1 -o tests/c/test_abi tests/c/test_abi.c -Iinclude -I/usr/local/cuda/include \
	    -L$(PKG) -laes_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$(abspath $(PKG)):/usr/local/cuda/lib64

clean:
	rm -rf build tests/c/test_abi

.PHONY: all c-test clean
