# Builds paper_2502_12082_b200/libentmax_attn.so (the C-ABI library) for sm_100a only.
NVCC   ?= nvcc
ARCH   := -gencode arch=compute_100a,code=sm_100a
CFLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -Ipaper_2502_12082_b200/csrc \
          --expt-relaxed-constexpr
SRC    := paper_2502_12082_b200/csrc
OBJS   := build/entmax_attn.o build/simt.o build/sm100.o
LIB    := paper_2502_12082_b200/libentmax_attn.so

PROBE  := tests/probe/libprobe.so

all: $(LIB) $(PROBE)

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
.PHONY: all clean
