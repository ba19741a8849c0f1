# Top-level build: the sm_100a engine (product) and the oracle (test infrastructure).
all: engine oracle

engine:
	$(MAKE) -C paper_2503_11674_b200/csrc -j8
	$(MAKE) -C paper_2503_11674_b200/host

oracle:
	$(MAKE) -C oracle all

clean:
	$(MAKE) -C paper_2503_11674_b200/csrc clean
	$(MAKE) -C oracle clean

.PHONY: all engine oracle clean
