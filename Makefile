# Top-level build: product library (nvcc, sm_100a) + CPU oracle (g++, test infrastructure).
all: gpu oracle

gpu:
	$(MAKE) -C paper_1704_06967_b200/csrc

oracle:
	$(MAKE) -C oracle

clean:
	$(MAKE) -C paper_1704_06967_b200/csrc clean
	$(MAKE) -C oracle clean

.PHONY: all gpu oracle clean
