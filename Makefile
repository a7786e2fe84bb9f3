# Builds paper_2502_12082_b200/libentmax_attn.so (the C-ABI library) for sm_100a only.
NVCC   ?= nvcc
ARCH   := -gencode arch=compute_100a,code=sm_100a
CFLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -Ipaper_2502_12082_b200/csrc \
          --expt-relaxed-constexpr
SRC    := paper_2502_12082_b200/csrc
OBJS   := build/entmax_attn.o build/simt.o build/sm100.o build/rowwise.o
LIB    := paper_2502_12082_b200/libentmax_attn.so

PROBE  := tests/probe/libprobe.so

TRACE  := tests/probe/libentmax_trace.so

all: $(LIB) $(PROBE)

trace: $(TRACE)

trace-nold: tests/probe/libentmax_trace_nold.so

tests/probe/libentmax_trace_nold.so: $(wildcard $(SRC)/*.cu $(SRC)/*.cuh $(SRC)/*.h) tests/probe/trace_api.cu
	$(NVCC) $(ARCH) $(CFLAGS) -DENTMAX_TRACE -DENTMAX_TRACE_NOLD -rdc=true -shared -o $@ $(SRC)/entmax_attn.cu $(SRC)/simt.cu $(SRC)/sm100.cu $(SRC)/rowwise.cu tests/probe/trace_api.cu

$(TRACE): $(wildcard $(SRC)/*.cu $(SRC)/*.cuh $(SRC)/*.h) tests/probe/trace_api.cu
	$(NVCC) $(ARCH) $(CFLAGS) -DENTMAX_TRACE -rdc=true -shared -o $@ $(SRC)/entmax_attn.cu $(SRC)/simt.cu $(SRC)/sm100.cu $(SRC)/rowwise.cu tests/probe/trace_api.cu

$(PROBE): tests/probe/probe.cu $(SRC)/sm100_ptx.cuh $(SRC)/tmap.h
	$(NVCC) $(ARCH) $(CFLAGS) -shared -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^

build/%.o: $(SRC)/%.cu
	@mkdir -p build
	$(NVCC) $(ARCH) $(CFLAGS) $(EXTRA) -MMD -MP -c -o $@ $<

clean:
	rm -rf build $(LIB) $(PROBE)

-include build/*.d
.PHONY: all clean trace
