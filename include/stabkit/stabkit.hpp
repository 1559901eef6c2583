// stabkit/stabkit.hpp -- umbrella header of the B200 host API.
#pragma once
#include "stabkit/bitvec.hpp"
#include "stabkit/circuit.hpp"
#include "stabkit/device.hpp"
#include "stabkit/engine.hpp"
#include "stabkit/error.hpp"
#include "stabkit/grouping.hpp"
#include "stabkit/pauli.hpp"
#include "stabkit/pbc.hpp"
#include "stabkit/rng.hpp"
#include "stabkit/sharded.hpp"
#include "stabkit/tableau.hpp"
