// ptrom_oracle_rom.hpp — CPU ORACLE (test infrastructure only), PTROM part (filled in later).
#pragma once
#include "ptrom_oracle_tree.hpp"
