# Build of the in-tree sm_100a library and the CPU oracle.
#   make            -> paper_2605_30218_b200/lib/libmargingate.so + oracle/liboracle.so
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr \
             -Xptxas -v -Iinclude
CSRC      := paper_2605_30218_b200/csrc
SRCS      := $(CSRC)/gemm.cu $(CSRC)/elementwise.cu $(CSRC)/attention.cu $(CSRC)/control.cu $(CSRC)/engine.cu \
             $(CSRC)/capi_debug.cu
BUILD     := build
OBJS      := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(SRCS))
LIB       := paper_2605_30218_b200/lib/libmargingate.so
HDRS      := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh include/*.h)

all: $(LIB) oracle/liboracle.so examples/mg_decode

# a plain C client of the C ABI (no Python / torch): caller-owned cudaMalloc buffers
examples/mg_decode: examples/mg_decode.c include/mg.h $(LIB)
	gcc -O2 -std=c11 -Wall -Iinclude -I/usr/local/cuda/include -o $@ examples/mg_decode.c \
	    -Lpaper_2605_30218_b200/lib -lmargingate -L/usr/local/cuda/lib64 -lcudart -lm \
	    -Wl,-rpath,'$$ORIGIN/../paper_2605_30218_b200/lib' -Wl,-rpath,/usr/local/cuda/lib64

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -ldl -lrt -lpthread

oracle/liboracle.so: oracle/mg_oracle.c oracle/mg_oracle.h
	gcc -O2 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math -Wall -o $@ oracle/mg_oracle.c -lm

clean:
	rm -rf $(BUILD) $(LIB) oracle/liboracle.so examples/mg_decode

.PHONY: all clean
